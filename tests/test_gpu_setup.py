"""Device preprocessing (csrc/gridlp_setup.cu via the C ABI) against the host
restatement of the reference's permute / slice / transpose
(partition.py:262-319, sparse_kernels.py:27-58): bit-identical block CSR,
transpose and SELL-32 arrays."""

import numpy as np
import pytest
import torch

from conftest import golden_problem, load_npz

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2601_07628_b200 import GridTopology, build_layout, native  # noqa: E402
from paper_2601_07628_b200.blocks import (DeviceSetup, HostCsr, build_sell, permute_matrix,  # noqa: E402
                                          slice_blocks, transpose)

DEV = torch.device("cuda", 0)


def _problem_with_long_rows():
    from paper_2601_07628_b200 import LpProblem, SparseMatrix

    rng = np.random.default_rng(5)
    m, n = 3000, 2500
    lens = rng.integers(0, 40, m)
    lens[[5, 900, 2999]] = [700, 1500, 2400]
    rows = np.repeat(np.arange(m), lens)
    cols = np.concatenate([rng.choice(n, k, replace=False) for k in lens])
    A = SparseMatrix.from_coo(m, n, rows, cols, rng.standard_normal(len(rows)))
    return LpProblem(matrix=A, objective=np.ones(n), var_lower=np.zeros(n), var_upper=np.ones(n),
                     con_lower=-np.ones(m), con_upper=np.ones(m))


CASES = [("u1000", (1, 1)), ("u1000", (2, 2)), ("tall", (2, 3)), ("heavy", (1, 1)), ("heavy", (2, 2)),
         ("heavy", (3, 1))]


@pytest.mark.parametrize("name,grid", CASES)
def test_device_blocks_match_host(name, grid):
    p = _problem_with_long_rows() if name == "heavy" else golden_problem(load_npz("layouts.npz"), name + "_")
    lay = build_layout(p, grid[0] * grid[1], grid=GridTopology(*grid), seed=3)
    host = slice_blocks(permute_matrix(p.matrix, lay), lay)
    setup = DeviceSetup(p, lay, DEV)
    for (i, j), hb in host.items():
        a = setup.block(i, j)
        assert a.nnz == hb.nnz
        np.testing.assert_array_equal(a.ptr.cpu().numpy(), hb.ptr)
        np.testing.assert_array_equal(a.col[: a.nnz].cpu().numpy(), hb.col)
        np.testing.assert_array_equal(a.val[: a.nnz].cpu().numpy(), hb.val)
        ht = transpose(hb)
        at = setup.transpose(a)
        np.testing.assert_array_equal(at.ptr.cpu().numpy(), ht.ptr)
        np.testing.assert_array_equal(at.col[: at.nnz].cpu().numpy(), ht.col)
        np.testing.assert_array_equal(at.val[: at.nnz].cpu().numpy(), ht.val)
        for dev_csr, host_csr in ((a, hb), (at, ht)):
            want = build_sell(host_csr, 512)
            got = setup.sell(dev_csr, 512)
            total = int(want["slice_off"][-1])
            np.testing.assert_array_equal(got["slice_off"].cpu().numpy(), want["slice_off"])
            np.testing.assert_array_equal(got["lane_info"].cpu().numpy()[: len(want["lane_info"])],
                                          want["lane_info"])
            np.testing.assert_array_equal(got["cols"][:total].cpu().numpy(), want["cols"][:total])
            np.testing.assert_array_equal(got["vals"][:total].cpu().numpy(), want["vals"][:total])
            np.testing.assert_array_equal(got["long_rows"].cpu().numpy(), want["long_rows"])
            np.testing.assert_array_equal(got["long_ptr"].cpu().numpy(), want["long_ptr"])
            hn = int(want["long_ptr"][-1])
            np.testing.assert_array_equal(got["long_cols"][:hn].cpu().numpy(), want["long_cols"][:hn])
            np.testing.assert_array_equal(got["long_vals"][:hn].cpu().numpy(), want["long_vals"][:hn])


def test_device_and_host_setup_solve_identically(golden_cfg1):
    from paper_2601_07628_b200 import SolverConfig
    from paper_2601_07628_b200.api import _solve

    p = golden_problem(golden_cfg1)
    cfg = SolverConfig(tolerance=1e-4, seed=0, n_procs=4, grid=(2, 2))
    a = _solve(p, cfg, engine_overrides={"device_setup": True, "first_touch_cols": False})
    b = _solve(p, cfg, engine_overrides={"device_setup": False, "first_touch_cols": False})
    np.testing.assert_array_equal(a.x, b.x)
    np.testing.assert_array_equal(a.y, b.y)
    assert a.layout == b.layout and a.counters == b.counters


def test_device_permute_matches_host():
    from paper_2601_07628_b200.blocks import DeviceCsrArrays, inverse_order, length_order, permute_csr

    rng = np.random.default_rng(5)
    m, n = 700, 900
    lens = rng.integers(0, 40, m)
    ptr = np.concatenate([[0], np.cumsum(lens)])
    col = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in lens]).astype(np.int64)
    val = rng.standard_normal(len(col))
    h = HostCsr(m, n, ptr, col, val)
    order = length_order(lens)
    label = inverse_order(rng.permutation(n))
    want = permute_csr(h, order, label)
    setup = DeviceSetup.__new__(DeviceSetup)
    setup.lib, setup.device = native.load(), DEV
    wsb = int(setup.lib._lib.gridlp_setup_workspace_bytes(len(col) + 64, m + 64))
    setup.ws, setup.ws_bytes = torch.empty(wsb, dtype=torch.uint8, device=DEV), wsb
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(DEV)  # noqa: E731
    a = DeviceCsrArrays(m, n, len(col), t(ptr, np.int32), t(np.concatenate([col, np.zeros(8)]), np.int32),
                        t(np.concatenate([val, np.zeros(8)]), np.float64))
    got = setup.permute(a, t(order, np.int32), t(label, np.int32))
    np.testing.assert_array_equal(got.ptr.cpu().numpy(), want.ptr)
    np.testing.assert_array_equal(got.col[: len(col)].cpu().numpy(), want.col)
    np.testing.assert_array_equal(got.val[: len(col)].cpu().numpy(), want.val)


@pytest.mark.parametrize("grid", [(1, 1), (2, 3)])
def test_sorted_internal_order_solves_like_natural(grid):
    """The internal length-sorted order only permutes storage: same status,
    iterations and restarts, and x / y equal up to reduction-order rounding."""
    from paper_2601_07628_b200 import GeneratorSpec, SolverConfig, generate
    from paper_2601_07628_b200.api import _solve

    p = generate(GeneratorSpec(kind="uniform_random", num_rows=600, num_cols=900, nnz_target=9000,
                               inequality_fraction=0.3, seed=4))
    cfg = SolverConfig(tolerance=1e-6, seed=4, n_procs=grid[0] * grid[1], grid=grid)
    a = _solve(p, cfg, engine_overrides={"sorted_order": True})
    b = _solve(p, cfg, engine_overrides={"sorted_order": False})
    assert (a.status, a.iterations, a.restarts) == (b.status, b.iterations, b.restarts)
    np.testing.assert_allclose(a.x, b.x, rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(a.y, b.y, rtol=1e-9, atol=1e-9)


def test_staged_upload_converts_and_matches():
    from paper_2601_07628_b200.blocks import STAGING_BYTES, upload

    rng = np.random.default_rng(0)
    big = STAGING_BYTES // 4 * 2 + 12345            # three chunks of int32
    cols = rng.integers(0, 2 ** 31 - 1, big)          # int64 source
    got = upload(cols, np.int32, DEV)
    assert got.dtype == torch.int32
    np.testing.assert_array_equal(got.cpu().numpy(), cols.astype(np.int32))
    vals = rng.standard_normal(STAGING_BYTES // 8 + 7)
    np.testing.assert_array_equal(upload(vals, np.float64, DEV).cpu().numpy(), vals)
    assert upload(np.zeros(0), np.float64, DEV).numel() == 0


def test_layout_autotune_choices_solve_identically():
    """The engine's timed layout choices (light_row_max per block, sorted vs
    layout order) change kernel paths only: a problem with rows in (128, 512]
    and longer solves bit for bit like every fixed choice."""
    from paper_2601_07628_b200 import GeneratorSpec, SolverConfig, generate
    from paper_2601_07628_b200.api import _solve
    from paper_2601_07628_b200.synth import McfSpec, generate_mcf

    p = generate_mcf(McfSpec(num_nodes=40, num_arcs=1200, num_commodities=300, seed=2),
                     torch.device("cuda", 0)).to_problem("mcf_small")
    cfg = SolverConfig(tolerance=1e-4, seed=1, max_iterations=640, permutation="none")
    auto = _solve(p, cfg)
    for over in ({"light_row_max": 128, "sorted_order": True}, {"light_row_max": 512, "sorted_order": False},
                 {"light_row_max": 256, "sorted_order": True}):
        r = _solve(p, cfg, engine_overrides=over)
        assert (r.status, r.iterations, r.restarts) == (auto.status, auto.iterations, auto.restarts)
        if over["sorted_order"] == (auto.timings.get("layout_order") == "sorted"):
            # same order: products bit-identical and canonical reductions -> everything equal
            np.testing.assert_array_equal(r.x, auto.x)
            np.testing.assert_array_equal(r.y, auto.y)
            assert r.report == auto.report
        else:   # another order sums the column-side reductions in another order (ulp level)
            np.testing.assert_allclose(r.x, auto.x, rtol=1e-9, atol=1e-9)
            np.testing.assert_allclose(r.y, auto.y, rtol=1e-9, atol=1e-9)
    q = generate(GeneratorSpec(kind="uniform_random", num_rows=300, num_cols=500, nnz_target=3000, seed=4))
    a = _solve(q, SolverConfig(tolerance=1e-6, seed=4))
    b = _solve(q, SolverConfig(tolerance=1e-6, seed=4), engine_overrides={"light_row_max": 128, "sorted_order": True})
    np.testing.assert_array_equal(a.x, b.x)


@pytest.mark.parametrize("over", [{"column_bands": 3, "sorted_order": False},
                                  {"column_bands": 3, "sorted_order": True},
                                  {"column_bands": 2, "light_row_max": 8, "exact_row_max": 32, "sorted_order": False},
                                  {"column_bands": 4, "light_row_max": 8, "exact_row_max": 32, "sorted_order": True}])
def test_column_bands_solve_identically(golden_cfg1, over):
    """Column-banded blocks (forced) solve bit for bit like unbanded ones,
    on the virtual grid and with row classes that put chunked rows in play."""
    from paper_2601_07628_b200 import SolverConfig
    from paper_2601_07628_b200.api import _solve

    p = golden_problem(golden_cfg1)
    base = {k: v for k, v in over.items() if k != "column_bands"}
    for grid in ((1, 1), (2, 2)):
        cfg = SolverConfig(tolerance=1e-6, seed=0, n_procs=grid[0] * grid[1], grid=grid, max_iterations=2048)
        a = _solve(p, cfg, engine_overrides=dict(base, column_bands=1))
        b = _solve(p, cfg, engine_overrides=over)
        assert (a.status, a.iterations, a.restarts) == (b.status, b.iterations, b.restarts)
        np.testing.assert_array_equal(a.x, b.x)
        np.testing.assert_array_equal(a.y, b.y)
        assert a.report == b.report


def test_order_choice_is_deterministic_and_structural():
    """sorted_order=None picks the order from the matrix alone: the same
    choice on every prepare; random rows keep the length-class order, a
    block-structured multi-commodity flow LP keeps its layout order."""
    from paper_2601_07628_b200 import GeneratorSpec, SolverConfig, generate
    from paper_2601_07628_b200.api import prepare
    from paper_2601_07628_b200.synth import McfSpec, generate_mcf

    mcf = generate_mcf(McfSpec(num_nodes=200, num_arcs=4000, num_commodities=60, seed=3),
                       torch.device("cuda", 0)).to_problem("mcf")
    rnd = generate(GeneratorSpec(kind="uniform_random", num_rows=20000, num_cols=40000, nnz_target=200000, seed=3))
    cfg = SolverConfig(tolerance=1e-4, seed=0, permutation="none")
    picks = {}
    for name, p in (("mcf", mcf), ("random", rnd)):
        got = [prepare(p, cfg)[0].choices["order"] for _ in range(2)]
        assert got[0] == got[1], name
        picks[name] = got[0]
    assert picks == {"mcf": "layout", "random": "sorted"}
