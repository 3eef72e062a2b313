"""On-device Ruiz + Pock-Chambolle scaling (scaling.py) against its numpy
restatement (oracle/scaling_oracle.py), and scaled solves against the
unscaled CPU oracle of the reference algorithm."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import pdhg_oracle, scaling_oracle  # noqa: E402
from paper_2601_07628_b200 import GeneratorSpec, SolverConfig, generate, solve  # noqa: E402
from paper_2601_07628_b200.problem import LpProblem, SparseMatrix  # noqa: E402
from paper_2601_07628_b200.scaling import scale_problem  # noqa: E402

DEV = torch.device("cuda", 0)


def _badly_scaled(seed, m=300, n=500, nnz=3000):
    """The reference generator's LP with rows and columns rescaled by
    10^U[-2, 2] (the same LP up to a diagonal change of variables)."""
    p = generate(GeneratorSpec(kind="uniform_random", num_rows=m, num_cols=n, nnz_target=nnz,
                               inequality_fraction=0.3, seed=seed))
    rng = np.random.default_rng(seed)
    r = 10.0 ** rng.uniform(-2, 2, m)
    c = 10.0 ** rng.uniform(-2, 2, n)
    A = p.matrix
    rows = np.repeat(np.arange(m), np.diff(A.row_offsets))
    val = A.values * r[rows] * c[A.col_indices]
    return LpProblem(SparseMatrix(m, n, A.row_offsets, A.col_indices, val), p.objective * c, p.var_lower / c,
                     p.var_upper / c, p.con_lower * r, p.con_upper * r), p


@pytest.mark.parametrize("mode", ["ruiz", "pock_chambolle", "ruiz+pock_chambolle"])
def test_scaling_bitwise(mode):
    p, _ = _badly_scaled(1)
    got = scale_problem(p, mode, 10, DEV)
    A = p.matrix
    val, dr, dc = scaling_oracle.scale(A.row_offsets, A.col_indices, A.values, A.num_rows, A.num_cols, mode, 10)
    np.testing.assert_array_equal(got.row_scale, dr)
    np.testing.assert_array_equal(got.col_scale, dc)
    np.testing.assert_array_equal(got.problem.matrix.values, val)
    np.testing.assert_array_equal(got.problem.objective, p.objective * dc)
    np.testing.assert_array_equal(got.problem.con_upper, p.con_upper * dr)
    np.testing.assert_array_equal(got.problem.var_upper, p.var_upper / dc)
    if mode == "ruiz":                     # Ruiz equilibrates: every row max close to 1
        absv = np.abs(got.problem.matrix.values)
        rows = np.repeat(np.arange(A.num_rows), np.diff(A.row_offsets))
        rmax = np.zeros(A.num_rows)
        np.maximum.at(rmax, rows, absv)
        assert np.all(rmax[rmax > 0] > 0.3) and np.all(rmax < 3.0)


def test_scaled_solve_matches_unscaled_optimum_and_needs_fewer_iterations():
    """The badly scaled LP p is a diagonal change of variables of the
    generator's LP q, so both have the same optimal objective: the unscaled
    reference algorithm stalls on p (iteration limit), the scaled solve of p
    reaches q's optimum."""
    p, q = _badly_scaled(2)
    base = dict(tolerance=1e-6, seed=2, max_iterations=100_000)
    plain = pdhg_oracle.oracle_solve(p, **base)
    well = pdhg_oracle.oracle_solve(q, **base)
    assert well.status == "optimal"
    got = solve(p, SolverConfig(**base, scaling="ruiz+pock_chambolle"))
    assert got.status == "optimal"
    assert abs(got.objective - well.objective) <= 1e-4 * max(1.0, abs(well.objective))
    assert got.iterations < plain.iterations
    # x, y come back in the original space: primal feasibility of the original LP
    ax = p.matrix.to_dense() @ got.x
    scale = 1.0 + np.max(np.abs(np.concatenate([p.con_lower, p.con_upper])))
    assert np.max(np.maximum(ax - p.con_upper, 0) + np.maximum(p.con_lower - ax, 0)) <= 1e-3 * scale
    assert np.all(got.x >= p.var_lower - 1e-9) and np.all(got.x <= p.var_upper + 1e-9)


def test_mps_instances_solve_like_reference():
    """MPS ingestion end to end: the reference CLI's toy instance solves to
    its known objective -8.0 (reference tests/test_cli.py:17-29), and each
    parsed golden case matches the CPU oracle's status and objective."""
    from conftest import load_json
    from paper_2601_07628_b200 import parse_mps

    cases = load_json("mps.json")["cases"]
    toy = solve(parse_mps(cases["toy3x2"]["text"]), SolverConfig(tolerance=1e-8))
    assert toy.status == "optimal" and abs(toy.objective - (-8.0)) <= 1e-6
    for name in ("toy3x2", "max_free"):
        p = parse_mps(cases[name]["text"])
        got = solve(p, SolverConfig(tolerance=1e-7, max_iterations=100_000))
        want = pdhg_oracle.oracle_solve(p, tolerance=1e-7, max_iterations=100_000)
        assert got.status == want.status
        assert (got.iterations, got.restarts) == (want.iterations, want.restarts)
        assert abs(got.objective - want.objective) <= 1e-6 * max(1.0, abs(want.objective))


def _host_rp(p, x):
    A = p.matrix
    rows = np.repeat(np.arange(A.num_rows), np.diff(A.row_offsets))
    ax = np.zeros(A.num_rows)
    np.add.at(ax, rows, A.values * x[A.col_indices])
    rv = np.maximum(ax - p.con_upper, 0.0) - np.maximum(p.con_lower - ax, 0.0)
    b = np.concatenate([p.con_lower, p.con_upper])
    return float(np.linalg.norm(rv)) / (1.0 + float(np.linalg.norm(b[np.isfinite(b)])))


@pytest.mark.parametrize("seed", [3, 4])
def test_scaled_solve_reports_original_kkt_and_matches_unscaled_oracle(seed):
    """SolverConfig.scaling: termination and the report are evaluated on the
    ORIGINAL LP (reference evaluate_kkt, pdhg_engine.py:310-346, at x = Dc x~,
    y = Dr y~). On a well-conditioned LP the scaled solve reaches the unscaled
    reference algorithm's status and objective to 1e-6 relative (both to a
    tight tolerance), and its reported primal residual / objective are those
    of the returned original-space x."""
    q = generate(GeneratorSpec(kind="uniform_random", num_rows=400, num_cols=700, nnz_target=5000,
                               inequality_fraction=0.3, seed=seed))
    base = dict(tolerance=1e-9, seed=seed, max_iterations=400_000)
    want = pdhg_oracle.oracle_solve(q, **base)
    got = solve(q, SolverConfig(**base, scaling="ruiz+pock_chambolle"))
    assert got.status == want.status == "optimal"
    assert abs(got.objective - want.objective) <= 1e-6 * max(1.0, abs(want.objective))
    rp = _host_rp(q, got.x)
    assert abs(got.report.r_primal - rp) <= 1e-6 * max(rp, 1e-300) + 1e-15
    assert got.report.overall <= 1e-9
    cx = float(np.dot(q.objective, got.x))
    assert abs(got.report.obj_primal - cx) <= 1e-9 * max(1.0, abs(cx))
    assert got.timings["scaling_s"] > 0


def test_scaled_solve_on_a_grid_matches_unscaled_oracle():
    """Scaling on a 2x2 virtual grid: the KKT scale vectors follow each grid
    band's internal order (engine ColState / RowState.scale), so the report
    is still the original LP's and the optimum the unscaled oracle's."""
    q = generate(GeneratorSpec(kind="uniform_random", num_rows=500, num_cols=800, nnz_target=6000,
                               inequality_fraction=0.3, seed=9))
    base = dict(tolerance=1e-9, seed=9, max_iterations=400_000)
    want = pdhg_oracle.oracle_solve(q, **base)
    got = solve(q, SolverConfig(**base, n_procs=4, grid=(2, 2), scaling="ruiz+pock_chambolle"))
    assert got.status == want.status == "optimal"
    assert abs(got.objective - want.objective) <= 1e-6 * max(1.0, abs(want.objective))
    rp = _host_rp(q, got.x)
    assert abs(got.report.r_primal - rp) <= 1e-6 * max(rp, 1e-300) + 1e-15


def test_scaling_refuses_band_problems():
    """A band problem has no global matrix to equilibrate (its blocks are
    generated per device): SolverConfig.scaling is refused up front."""
    from paper_2601_07628_b200 import synth

    p = synth.BandProblem(synth.PlantedBands(synth.PlantedSpec(100, 200, 4)), "planted")
    with pytest.raises(ValueError, match="band problems"):
        solve(p, SolverConfig(scaling="ruiz", permutation="none", partitioning="uniform"))
