"""Pins the PACKAGE's layout code (paper_2601_07628_b200/layout.py: the
vectorised Fisher-Yates of block_random_permutation, the searchsorted nnz
cuts, select_grid, layout_summary) to the reference's own layouts
(tests/golden/layouts.*, produced by tests/golden/make_golden.py importing
/root/reference/pkg/src/gridlp/partition.py:131-378). Integer work, so the
bar is bit-exact. test_oracle_golden.py pins the oracle; this file pins the
product."""

import numpy as np

from conftest import golden_problem, load_json, load_npz
from paper_2601_07628_b200 import layout as L


def test_build_layout_matches_reference_layouts():
    z = load_npz("layouts.npz")
    meta = load_json("layouts.json")
    probs = {}
    assert len(meta) == 168
    for m in meta:
        p = probs.setdefault(m["problem"], golden_problem(z, m["problem"] + "_"))
        grid = None if m["grid"] is None else L.GridTopology(*m["grid"])
        lay = L.build_layout(p, m["procs"], block_size=m["block_size"], seed=m["seed"],
                             permutation=m["permutation"], partitioning=m["partitioning"], grid=grid)
        t = m["id"]
        assert [lay.topology.rows, lay.topology.cols] == m["topology"], m
        np.testing.assert_array_equal(lay.perm.row_perm, z[f"L{t}_row_perm"], err_msg=str(m))
        np.testing.assert_array_equal(lay.perm.col_perm, z[f"L{t}_col_perm"], err_msg=str(m))
        np.testing.assert_array_equal(lay.row_cuts, z[f"L{t}_row_cuts"], err_msg=str(m))
        np.testing.assert_array_equal(lay.col_cuts, z[f"L{t}_col_cuts"], err_msg=str(m))
        assert L.layout_summary(p, lay) == m["summary"], m


def test_select_grid_matches_reference():
    z = load_npz("layouts.npz")
    cases = z["select_grid"]
    assert len(cases) == 180
    for m, n, procs, r, c in cases:
        g = L.select_grid(int(m), int(n), int(procs))
        assert (g.rows, g.cols) == (r, c), (m, n, procs)


def test_unpermute_inverts_layout():
    z = load_npz("layouts.npz")
    p = golden_problem(z, "u300_")
    lay = L.build_layout(p, 4, grid=L.GridTopology(2, 2), seed=1)
    np.testing.assert_array_equal(lay.perm.row_perm, z["B_row_perm"])
    x = np.arange(p.matrix.num_cols, dtype=np.float64)
    y = np.arange(p.matrix.num_rows, dtype=np.float64)
    xp, yp = x[lay.perm.col_perm], y[lay.perm.row_perm]
    xb = [xp[lay.col_cuts[j]:lay.col_cuts[j + 1]] for j in range(2)]
    yb = [yp[lay.row_cuts[i]:lay.row_cuts[i + 1]] for i in range(2)]
    xo, yo = L.unpermute_solution(lay, xb, yb)
    np.testing.assert_array_equal(xo, x)
    np.testing.assert_array_equal(yo, y)
