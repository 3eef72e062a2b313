"""Pins the CPU oracle (oracle/pdhg_oracle.py) to the reference's own outputs
(tests/golden/*, produced by tests/golden/make_golden.py importing
/root/reference/pkg/src/gridlp). Bit-exact: the oracle restates the same
numpy/scipy arithmetic in the same order."""

import math

import numpy as np
import pytest

from conftest import golden_problem, load_json, load_npz
from oracle import pdhg_oracle as O


def _cfg(meta):
    c = dict(meta["cfg"])
    if c.get("grid") is not None:
        c["grid"] = tuple(c["grid"])
    return c


class TestSpmvPins:
    def test_scipy_products_match_reference(self):
        z = load_npz("spmv.npz")
        for t in range(int(z["ncases"])):
            a = O.as_csr(type("M", (), dict(num_rows=z[f"c{t}_m"], num_cols=z[f"c{t}_n"],
                                            row_offsets=z[f"c{t}_ptr"], col_indices=z[f"c{t}_col"],
                                            values=z[f"c{t}_val"]))())
            np.testing.assert_array_equal(O.seq_spmv(a, z[f"c{t}_x"]), z[f"c{t}_ax"])
            at = O.csr_transpose(a)
            np.testing.assert_array_equal(at.indptr, z[f"c{t}_tptr"])
            np.testing.assert_array_equal(at.indices, z[f"c{t}_tcol"])
            np.testing.assert_array_equal(O.seq_spmv(at, z[f"c{t}_y"]), z[f"c{t}_aty"])

    def test_sequential_loop_definition(self):
        z = load_npz("spmv.npz")
        ptr, col, val, x = z["c0_ptr"], z["c0_col"], z["c0_val"], z["c0_x"]
        out = np.zeros(len(ptr) - 1)
        for i in range(len(ptr) - 1):
            acc = 0.0
            for k in range(ptr[i], ptr[i + 1]):
                acc += val[k] * x[col[k]]
            out[i] = acc
        np.testing.assert_array_equal(out, z["c0_ax"])


class TestLayoutPins:
    def test_layouts(self):
        z = load_npz("layouts.npz")
        meta = load_json("layouts.json")
        probs = {}
        for m in meta:
            p = probs.setdefault(m["problem"], golden_problem(z, m["problem"] + "_"))
            a = O.as_csr(p.matrix)
            lay = O.make_layout(a, m["procs"], m["block_size"], m["seed"], m["permutation"],
                                m["partitioning"], None if m["grid"] is None else tuple(m["grid"]))
            t = m["id"]
            assert [lay.rows, lay.cols] == m["topology"]
            np.testing.assert_array_equal(lay.row_perm, z[f"L{t}_row_perm"])
            np.testing.assert_array_equal(lay.col_perm, z[f"L{t}_col_perm"])
            np.testing.assert_array_equal(lay.row_cuts, z[f"L{t}_row_cuts"])
            np.testing.assert_array_equal(lay.col_cuts, z[f"L{t}_col_cuts"])
            assert O.layout_summary(a, lay) == m["summary"]

    def test_select_grid(self):
        z = load_npz("layouts.npz")
        for m, n, procs, r, c in z["select_grid"]:
            assert O.grid_shape(int(m), int(n), int(procs)) == (r, c)

    def test_blocks(self):
        z = load_npz("layouts.npz")
        p = golden_problem(z, "u300_")
        a = O.as_csr(p.matrix)
        lay = O.make_layout(a, 4, grid=(2, 2), seed=1)
        np.testing.assert_array_equal(lay.row_perm, z["B_row_perm"])
        pa = O.permute_csr(a, lay)
        for i in range(2):
            for j in range(2):
                blk = O.take_block(pa, lay.row_cuts[i], lay.row_cuts[i + 1],
                                   lay.col_cuts[j], lay.col_cuts[j + 1])
                np.testing.assert_array_equal(blk.indptr, z[f"B{i}{j}_ptr"])
                np.testing.assert_array_equal(blk.indices, z[f"B{i}{j}_col"])
                np.testing.assert_array_equal(blk.data, z[f"B{i}{j}_val"])
                t = O.csr_transpose(blk)
                np.testing.assert_array_equal(t.indptr, z[f"B{i}{j}_tptr"])
                np.testing.assert_array_equal(t.indices, z[f"B{i}{j}_tcol"])
                np.testing.assert_array_equal(t.data, z[f"B{i}{j}_tval"])


class TestSolvePins:
    def test_cfg1_bitwise(self, golden_cfg1):
        z = golden_cfg1
        p = golden_problem(z)
        r = O.oracle_solve(p, trace_at=list(z["trace_iters"]), tolerance=1e-4, seed=0)
        assert (r.status, r.iterations, r.restarts) == ("optimal", int(z["iterations"]),
                                                         int(z["restarts"]))
        assert r.objective == float(z["result_objective"])
        np.testing.assert_array_equal(r.x, z["x"])
        np.testing.assert_array_equal(r.y, z["y"])
        for k, it in enumerate(z["trace_iters"]):
            np.testing.assert_array_equal(r.trace[int(it)][0], z["trace_x"][k])
            np.testing.assert_array_equal(r.trace[int(it)][1], z["trace_y"][k])
        np.testing.assert_array_equal(np.array(r.passes), z["passlog"])

    def test_cfg1_power_estimate(self, golden_cfg1):
        p = golden_problem(golden_cfg1)
        assert O.power_estimate(p, seed=0) == float(golden_cfg1["estimate"])

    def test_cfg1_fixed_eta(self, golden_cfg1):
        z = golden_cfg1
        p = golden_problem(z)
        r = O.oracle_solve(p, trace_at=list(z["fx_trace_iters"]), tolerance=1e-300, seed=0,
                           eta=0.05, restarts=False, max_iterations=512)
        for k, it in enumerate(z["fx_trace_iters"]):
            np.testing.assert_array_equal(r.trace[int(it)][0], z["fx_trace_x"][k])
            np.testing.assert_array_equal(r.trace[int(it)][1], z["fx_trace_y"][k])
        np.testing.assert_array_equal(r.x, z["fx_x"])

    @pytest.mark.parametrize("chunk", range(6))
    def test_solve_cases_bitwise(self, golden_solves, chunk):
        z, meta = golden_solves
        cases = [m for m in meta if "result" in m and "time_limit_seconds" not in m["cfg"]]
        for m in cases[chunk::6]:
            p = golden_problem(z, m["problem"] + "_")
            r = O.oracle_solve(p, **_cfg(m))
            exp = m["result"]
            t = m["id"]
            assert r.status == exp["status"], m
            assert r.iterations == exp["iterations"], m
            assert r.restarts == exp["restarts"], m
            np.testing.assert_array_equal(r.x, z[f"S{t}_x"])
            np.testing.assert_array_equal(r.y, z[f"S{t}_y"])
            for key, val in (("r_primal", r.r_primal), ("r_dual", r.r_dual), ("r_gap", r.r_gap),
                             ("obj_primal", r.obj_primal), ("obj_dual", r.obj_dual)):
                want = exp["kkt"][key]
                assert (val == want) or (math.isnan(val) and math.isnan(want)), (m, key)
            assert r.layout == exp["layout"]


def test_synth_oracle_instances_are_feasible_and_canonical():
    """The generator restatement: rows sorted and distinct, the planted
    point satisfies every bound, and the package's host hash equals it."""
    from oracle import synth_oracle
    from paper_2601_07628_b200.synth import host_u01, mcf_graph, McfSpec

    for inst in (synth_oracle.powerlaw(700, 900, 7000, seed=3), synth_oracle.mcf(15, 80, 4, seed=3)):
        ptr, col = inst["ptr"], inst["col"]
        for r in range(len(ptr) - 1):
            assert np.all(np.diff(col[ptr[r]:ptr[r + 1]]) > 0)
        import scipy.sparse as sp

        A = sp.csr_matrix((inst["val"], col, ptr), shape=(len(ptr) - 1, len(inst["x_hat"])))
        ax = A.dot(inst["x_hat"])
        assert np.all(ax >= inst["con_lo"]) and np.all(ax <= inst["con_hi"])
        assert np.all(inst["x_hat"] >= inst["var_lo"]) and np.all(inst["x_hat"] <= inst["var_hi"])
    idx = np.arange(1000)
    np.testing.assert_array_equal(host_u01(7, 3, idx), synth_oracle.u01(7, 3, idx))
    tail, head, *_ = mcf_graph(McfSpec(30, 500, 2, seed=4))
    assert np.all(tail != head)
