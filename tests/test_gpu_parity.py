"""Parity of the sm_100a path (through the C ABI) with the reference.

Bars (stated per test):
  * sparse products with rows <= exact_row_max: BIT-IDENTICAL to scipy's
    csr_matvec (the reference kernel); longer rows: <= 1e-12 relative;
  * every epilogue op: BIT-IDENTICAL to the reference's numpy expression,
    including NaN / inf / signed-zero cases;
  * fixed-step (eta given) restart-free trajectories: BIT-IDENTICAL iterates
    at every checkpoint (the device reproduces every rounding);
  * full solves: identical status / iterations / restarts; objective and KKT
    residuals within 1e-6 relative (north-star bar) and iterates within
    1e-9 relative in max-norm. Only the norm/dot reductions use a different
    (deterministic, tree) summation order than numpy's ddot.
"""

import math

import numpy as np
import pytest
import torch

from conftest import golden_problem, load_json, load_npz
from host_ops import HostOps

pytestmark = pytest.mark.gpu

cuda = pytest.importorskip("torch").cuda
if not cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2601_07628_b200 import SolverConfig, native, solve, reference_solve  # noqa: E402
from paper_2601_07628_b200.blocks import DeviceCsr, HostCsr  # noqa: E402
from paper_2601_07628_b200.engine import ColState, RowState  # noqa: E402
from paper_2601_07628_b200.ops import CudaOps, Fused, Parts  # noqa: E402

DEV = torch.device("cuda", 0)


@pytest.fixture(scope="module")
def ops():
    return CudaOps(DEV, 1 << 16, 16)


def host_csr(m, n, ptr, col, val):
    return HostCsr(int(m), int(n), np.asarray(ptr, np.int64), np.asarray(col, np.int64),
                   np.asarray(val, np.float64))


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=DEV)


def test_library_is_loaded_from_tree():
    lib = native.load()
    assert lib.path == native.LIB_PATH
    sm, l2 = lib.device_info(0)
    assert sm >= 100 and l2 > 0


class TestProducts:
    def test_golden_spmv_bitwise(self, ops):
        z = load_npz("spmv.npz")
        for t in range(int(z["ncases"])):
            for tag, vec, want in (("", "x", "ax"), ("t", "y", "aty")):
                h = host_csr(z[f"c{t}_m"] if tag == "" else z[f"c{t}_n"],
                             z[f"c{t}_n"] if tag == "" else z[f"c{t}_m"],
                             z[f"c{t}_{tag}ptr"], z[f"c{t}_{tag}col"], z[f"c{t}_{tag}val"])
                A = DeviceCsr(h, DEV)
                out = torch.full((h.num_rows,), np.nan, dtype=torch.float64, device=DEV)
                ops.store(Fused(A, dev(z[f"c{t}_{vec}"])), out)
                np.testing.assert_array_equal(out.cpu().numpy(), z[f"c{t}_{want}"])

    @pytest.mark.parametrize("seed", range(3))
    def test_random_bitwise_and_long_rows(self, ops, seed):
        import scipy.sparse as sp

        rng = np.random.default_rng(seed)
        m, n = 3000, 5000
        lens = rng.integers(0, 60, m)
        lens[[7, 500, 1200, 2000, 2999]] = rng.integers(600, 5000, 5)   # long rows
        lens[7] = 4800                                                   # heavy (> 4096)
        lens[100:300] = 0
        ptr = np.concatenate([[0], np.cumsum(lens)])
        col = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in lens]).astype(np.int64)
        val = rng.standard_normal(len(col)) * 10.0 ** rng.integers(-6, 6, len(col))
        x = rng.standard_normal(n)
        h = host_csr(m, n, ptr, col, val)
        want = sp.csr_matrix((val, col, ptr), shape=(m, n)).dot(x)
        A = DeviceCsr(h, DEV)
        assert A.long_rows == np.count_nonzero(lens > 128)
        assert A.heavy_rows == np.count_nonzero(lens > 4096)
        out = torch.empty(m, dtype=torch.float64, device=DEV)
        ops.store(Fused(A, dev(x)), out)
        got = out.cpu().numpy()
        light = lens <= 4096
        np.testing.assert_array_equal(got[light], want[light])
        scale = np.abs(val[None, :]).max() * np.abs(x).max()
        if (~light).any():
            assert np.max(np.abs(got[~light] - want[~light])) <= 1e-12 * scale * lens.max()
        out2 = torch.empty_like(out)
        ops.store(Fused(A, dev(x)), out2)
        assert torch.equal(out, out2)          # deterministic

    def test_chunked_long_rows(self, ops):
        """Rows of up to ~200k entries split over many chunk CTAs: FP64
        tolerance vs scipy, bitwise reproducible across launches (the
        arrival counters reset themselves); light and long-exact rows still
        bit-exact, and fused reductions see every row exactly once."""
        import scipy.sparse as sp

        C = native.HEAVY_CHUNK
        rng = np.random.default_rng(7)
        m, n = 2000, 300_000
        lens = rng.integers(0, 30, m)
        lens[[0, 1, 5, 999, 1999]] = [200_000, C, C + 1, 7 * C + 5, 513]
        ptr = np.concatenate([[0], np.cumsum(lens)])
        col = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in lens]).astype(np.int64)
        val = rng.standard_normal(len(col))
        x = rng.standard_normal(n)
        h = host_csr(m, n, ptr, col, val)
        want = sp.csr_matrix((val, col, ptr), shape=(m, n)).dot(x)
        A = DeviceCsr(h, DEV)
        assert A.long_rows == 5 and A.heavy_rows == 2
        assert A.num_chunks == sum(-(-k // C) for k in lens[lens > 4096])
        outs = []
        for _ in range(3):
            out = torch.empty(m, dtype=torch.float64, device=DEV)
            ops.store(Fused(A, dev(x)), out)
            outs.append(out.cpu().numpy())
        assert all(np.array_equal(outs[0], o) for o in outs[1:])
        light = lens <= 4096
        np.testing.assert_array_equal(outs[0][light], want[light])
        for r in np.flatnonzero(~light):
            scale = np.sum(np.abs(val[ptr[r]:ptr[r + 1]] * x[col[ptr[r]:ptr[r + 1]]]))
            assert abs(outs[0][r] - want[r]) <= 1e-13 * scale
        assert torch.equal(A.dev["chunk_done"], torch.zeros_like(A.dev["chunk_done"]))
        # fused reduction: sum of squares of the outputs (power-iteration op)
        out = torch.empty(m, dtype=torch.float64, device=DEV)
        ops.store(Fused(A, dev(x)), out, slot=0)
        ssq = float(ops.read_slots(1)[0][0])
        assert abs(ssq - float(np.sum(outs[0] ** 2))) <= 1e-12 * float(np.sum(outs[0] ** 2))

    @pytest.mark.parametrize("light,exact", [(64, 4096), (0, 4096), (8, 8), (1, 65536), (512, 4096), (2048, 4096)])
    def test_row_classes_bitwise(self, ops, light, exact):
        """Every row up to exact_row_max is the sequential +0.0-seeded sum
        whichever class sums it (SELL lane, warp per row), including
        signed zeros, infinities and NaN."""
        import scipy.sparse as sp

        rng = np.random.default_rng(light + exact)
        m, n = 1500, 9000
        lens = rng.integers(0, 3000, m)
        lens[::7] = rng.integers(0, 20, len(lens[::7]))
        ptr = np.concatenate([[0], np.cumsum(lens)])
        col = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in lens]).astype(np.int64)
        val = rng.standard_normal(len(col)) * 10.0 ** rng.integers(-8, 8, len(col))
        x = rng.standard_normal(n)
        x[:4] = [np.inf, -np.inf, np.nan, -0.0]
        val[rng.choice(len(val), 50, replace=False)] = -0.0
        h = host_csr(m, n, ptr, col, val)
        with np.errstate(invalid="ignore"):
            want = sp.csr_matrix((val, col, ptr), shape=(m, n)).dot(x)
        A = DeviceCsr(h, DEV, exact_row_max=exact, light_row_max=light)
        out = torch.empty(m, dtype=torch.float64, device=DEV)
        ops.store(Fused(A, dev(x)), out)
        got = out.cpu().numpy()
        ok = lens <= exact
        np.testing.assert_array_equal(got[ok], want[ok])
        num = ok & ~np.isnan(want)         # NaN sign/payload is not IEEE-specified (x86 vs GPU default NaN)
        assert np.array_equal(np.signbit(got[num]), np.signbit(want[num]))

    @pytest.mark.parametrize("K,light,exact", [(3, 64, 4096), (4, 8, 64), (2, 0, 16)])
    def test_column_bands_bitwise(self, ops, K, light, exact):
        """BandedCsr (column bands chained through the carry buffer) ==
        the unbanded block bit for bit, with SELL, warp-per-row and chunked
        rows (the latter kept whole in the last band) and empty rows."""
        from paper_2601_07628_b200.blocks import BandedCsr, DeviceCsrArrays, split_column_bands

        rng = np.random.default_rng(K * 100 + light)
        m, n = 900, 5000
        lens = rng.integers(0, 300, m)
        lens[::5] = 0
        lens[3] = 2000
        ptr = np.concatenate([[0], np.cumsum(lens)])
        col = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in lens]).astype(np.int64)
        val = rng.standard_normal(len(col)) * 10.0 ** rng.integers(-8, 8, len(col))
        x = rng.standard_normal(n)
        h = host_csr(m, n, ptr, col, val)
        whole = DeviceCsr(h, DEV, exact_row_max=exact, light_row_max=light)
        want = torch.empty(m, dtype=torch.float64, device=DEV)
        ops.store(Fused(whole, dev(x)), want)
        arr = DeviceCsrArrays(m, n, len(col), torch.as_tensor(ptr.astype(np.int32), device=DEV),
                              torch.as_tensor(np.concatenate([col, np.zeros(8, np.int64)]).astype(np.int32), device=DEV),
                              dev(np.concatenate([val, np.zeros(8)])))
        cuts = [(k * n) // K for k in range(K + 1)]
        parts = split_column_bands(arr, cuts, exact)
        assert sum(p.nnz for p in parts) == len(col)
        bands = [DeviceCsr(host_csr(m, n, p.ptr.cpu().numpy(), p.col[:p.nnz].cpu().numpy(),
                                    p.val[:p.nnz].cpu().numpy()), DEV, exact_row_max=exact, light_row_max=light)
                 for p in parts]
        banded = BandedCsr(bands, cuts, DEV)
        cap = CudaOps(DEV, banded.slots() + whole.slots() + 8, 4)
        got = torch.empty(m, dtype=torch.float64, device=DEV)
        cap.store(Fused(banded, dev(x)), got)
        np.testing.assert_array_equal(got.cpu().numpy(), want.cpu().numpy())

    def test_parts_sum_ascending(self, ops):
        rng = np.random.default_rng(3)
        parts = [rng.standard_normal(777) * 10.0 ** rng.integers(-8, 8, 777) for _ in range(5)]
        out = torch.empty(777, dtype=torch.float64, device=DEV)
        ops.store(Parts([dev(p) for p in parts], 777), out)
        want = parts[0].copy()
        for p in parts[1:]:
            want += p
        np.testing.assert_array_equal(out.cpu().numpy(), want)


    def test_div_norm_equals_host_divisor(self, ops):
        """gridlp_op_div_norm (divisor sqrt(s_sq) read from a reduction slot
        on the device) == gridlp_op_div with the divisor computed on the host
        by math.sqrt, bit for bit (power iteration, sparse_kernels.py:92)."""
        rng = np.random.default_rng(11)
        s = rng.standard_normal(5003) * 10.0 ** rng.integers(-6, 6, 5003)
        src = dev(s)
        for sq in (2.0, 3.0e-7, 1.2345678901234567e11, float(np.dot(s, s))):
            ops.slots[5, 0] = sq
            a = torch.empty_like(src)
            b = torch.empty_like(src)
            ops.div_norm(src, a, 5)
            ops.div(src, b, math.sqrt(sq))
            np.testing.assert_array_equal(a.cpu().numpy(), b.cpu().numpy())
            np.testing.assert_array_equal(a.cpu().numpy(), s / math.sqrt(sq))


def _edge_vectors(rng, n):
    v = rng.standard_normal(n) * 10.0 ** rng.integers(-3, 3, n)
    special = [0.0, -0.0, np.inf, -np.inf, 1e-300, -1e308, 5.0]
    v[: len(special)] = special
    return v


class TestEpilogueOps:
    """Each op against the CPU double (numpy, reference order), bitwise."""

    def _states(self, rng, n, m, host):
        def mk(a):
            return torch.as_tensor(a.copy()) if host else dev(a)
        lo = rng.uniform(-2, 0, n)
        hi = lo + rng.uniform(0, 3, n)
        lo[:3], hi[3:6] = -np.inf, np.inf
        lo[6], hi[6] = 1.0, 1.0
        x = _edge_vectors(rng, n)
        x[10] = np.nan
        col = ColState(0, n, mk(rng.standard_normal(n)), mk(lo), mk(hi), mk(x), mk(np.zeros(n)),
                       mk(rng.standard_normal(n)), mk(np.zeros(n)), mk(np.zeros(n)), mk(np.zeros(n)))
        clo = rng.uniform(-2, 0, m)
        chi = clo + rng.uniform(0, 1, m)
        clo[:4], chi[2:7] = -np.inf, np.inf
        y = _edge_vectors(rng, m)
        y[9] = np.nan
        row = RowState(0, m, mk(clo), mk(chi), mk(y), mk(rng.standard_normal(m)), mk(np.zeros(m)),
                       mk(np.zeros(m)), mk(np.zeros(m)))
        return col, row

    @pytest.mark.parametrize("gamma,halpern", [(0.0, True), (0.5, True), (0.0, False)])
    def test_primal_dual_kkt_probe(self, ops, gamma, halpern):
        rng = np.random.default_rng(11)
        n, m = 2000, 1500
        sums_n = _edge_vectors(rng, n)
        sums_m = _edge_vectors(rng, m)
        hops = HostOps(None, 0, 16)
        results = []
        for host in (False, True):
            r2 = np.random.default_rng(5)
            col, row = self._states(r2, n, m, host)
            o = hops if host else ops
            mk = (lambda a: torch.as_tensor(a.copy())) if host else dev
            sn, sm_ = Parts([mk(sums_n)], n), Parts([mk(sums_m)], m)
            o.set_step(0.37, 1.9, gamma, 41)
            o.primal(sn, col, 3, halpern)
            o.dual(sm_, row, 3, halpern)
            ax = mk(np.zeros(m))
            o.kkt_rows(sm_, row, ax, 0)
            o.kkt_cols(sn, col, 1)
            dy = mk(np.zeros(m))
            o.probe(sm_, row, mk(sums_m[::-1].copy()), dy, 2)
            o.anchor(col.x, col.x0, 3)
            res = [t.cpu().numpy().copy() for t in (col.x, col.xbar, col.xpb, col.x0, row.y, ax, dy)]
            results.append((res, o.read_slots(4)))
        (gpu, gs), (cpu, cs) = results
        for a, b in zip(gpu, cpu):
            np.testing.assert_array_equal(a, b)
            np.testing.assert_array_equal(np.signbit(a), np.signbit(b))
        # reductions: same value up to summation order (NaN where numpy has NaN)
        for q, (a, b) in enumerate(zip(gs.ravel(), cs.ravel())):
            if math.isnan(b):
                assert math.isnan(a), q
            elif math.isinf(b):
                assert a == b, q
            else:
                assert abs(a - b) <= 1e-12 * max(1.0, abs(b)), (q, a, b)


class TestSolves:
    def test_fixed_eta_trajectory_bitwise(self, golden_cfg1):
        z = golden_cfg1

        class Keep(list):
            keep = set(int(t) for t in z["fx_trace_iters"])

        tr = Keep()
        r = reference_solve(golden_problem(z), SolverConfig(tolerance=1e-300, seed=0, eta=0.05,
                                                           restarts=False, max_iterations=512), trace=tr)
        assert [t for t, _, _ in tr] == [int(t) for t in z["fx_trace_iters"]]
        for k, (_, x, y) in enumerate(tr):
            np.testing.assert_array_equal(x, z["fx_trace_x"][k])
            np.testing.assert_array_equal(y, z["fx_trace_y"][k])
        np.testing.assert_array_equal(r.x, z["fx_x"])
        for a, b in zip([r.report.r_primal, r.report.r_dual, r.report.r_gap, r.report.obj_primal,
                         r.report.obj_dual], z["fx_kkt"]):
            assert abs(a - b) <= 1e-12 * max(1.0, abs(b))

    def test_graph_replay_equals_eager(self, golden_cfg1):
        from paper_2601_07628_b200.api import _solve

        p = golden_problem(golden_cfg1)
        cfg = SolverConfig(tolerance=1e-300, seed=0, eta=0.05, restarts=False, max_iterations=640)
        a = _solve(p, cfg, engine_overrides={"use_graphs": True})
        b = _solve(p, cfg, engine_overrides={"use_graphs": False})
        np.testing.assert_array_equal(a.x, b.x)
        np.testing.assert_array_equal(a.y, b.y)

    def test_cfg1_to_tolerance(self, golden_cfg1):
        z = golden_cfg1
        r = solve(golden_problem(z), SolverConfig(tolerance=1e-4, seed=0))
        assert (r.status, r.iterations, r.restarts) == ("optimal", int(z["iterations"]), int(z["restarts"]))
        ref = float(z["result_objective"])
        assert abs(r.objective - ref) <= 1e-6 * abs(ref)
        for a, b in zip([r.report.r_primal, r.report.r_dual, r.report.r_gap], z["kkt"][:3]):
            assert abs(a - b) <= 1e-6 * max(abs(b), 1e-12)
        for got, want in ((r.x, z["x"]), (r.y, z["y"])):
            assert np.max(np.abs(got - want)) <= 1e-9 * max(1.0, np.max(np.abs(want)))
        again = solve(golden_problem(z), SolverConfig(tolerance=1e-4, seed=0))
        np.testing.assert_array_equal(r.x, again.x)   # run-to-run deterministic

    @pytest.mark.parametrize("chunk", range(4))
    def test_golden_cases(self, golden_solves, chunk):
        z, meta = golden_solves
        for m in [m for m in meta if "result" in m][chunk::4]:
            cfg = dict(m["cfg"])
            if cfg.get("grid") is not None:
                cfg["grid"] = tuple(cfg["grid"])
            r = solve(golden_problem(z, m["problem"] + "_"), SolverConfig(**cfg))
            exp = m["result"]
            assert r.status == exp["status"], m["id"]
            assert r.iterations == exp["iterations"], m["id"]
            assert r.restarts == exp["restarts"], m["id"]
            assert r.counters == exp["counters"], m["id"]
            assert r.layout == exp["layout"], m["id"]
            if r.status in ("optimal", "iteration_limit"):
                want = exp["objective"]
                assert abs(r.objective - want) <= 1e-6 * max(1.0, abs(want)), m["id"]
                xr = z[f"S{m['id']}_x"]
                assert np.max(np.abs(r.x - xr), initial=0.0) <= 1e-6 * max(1.0, np.max(np.abs(xr), initial=0.0))


def test_pdhg_iterate_equals_op_by_op(golden_cfg1):
    """gridlp_pdhg_iterate (one C call for a chunk of iterations) launches
    the same primal/dual ops as the op-by-op loop: identical iterates and
    Halpern counter."""
    from paper_2601_07628_b200.api import prepare

    p = golden_problem(golden_cfg1)
    states = []
    for fused in (True, False):
        eng, _, eta, omega, _ = prepare(p, SolverConfig(seed=0), engine_overrides={"use_graphs": False})
        eng.start(eta, omega)
        eng.ops.set_step(eta / omega, eta * omega, 0.0, 0)
        (j, col), = eng.cols.items()
        (i, row), = eng.rows.items()
        if fused:
            eng.ops.iterate(eng.plan_primal[j][2], col, eng.plan_dual[i][2], row, 37, True)
        else:
            for t in range(37):
                eng.ops.primal(eng.plan_primal[j][2], col, t, True)
                eng.ops.dual(eng.plan_dual[i][2], row, t, True)
            eng.ops.step_advance(37)
        states.append((col.x.cpu().numpy(), row.y.cpu().numpy(), eng.ops.step.cpu().numpy()))
    for a, b in zip(*states):
        np.testing.assert_array_equal(a, b)
