"""Device generators (csrc/gridlp_gen.cu via synth.py) against their numpy
restatement (oracle/synth_oracle.py): bit-identical instances, then solves
of small generated LPs against the CPU oracle of the reference algorithm."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import pdhg_oracle, synth_oracle  # noqa: E402
from paper_2601_07628_b200 import SolverConfig, solve  # noqa: E402
from paper_2601_07628_b200.synth import McfSpec, PowerLawSpec, generate_mcf, generate_powerlaw  # noqa: E402

DEV = torch.device("cuda", 0)


def _same(dl, want):
    got = dict(ptr=dl.row_ptr, col=dl.cols, val=dl.vals, x_hat=dl.x_hat, c=dl.objective, var_lo=dl.var_lower,
               var_hi=dl.var_upper, con_lo=dl.con_lower, con_hi=dl.con_upper)
    for k, v in want.items():
        np.testing.assert_array_equal(got[k].cpu().numpy(), v, err_msg=k)


@pytest.mark.parametrize("m,n,nnz,seed", [(3000, 5000, 30000, 0), (500, 20000, 40000, 5), (4000, 300, 9000, 2)])
def test_powerlaw_bitwise(m, n, nnz, seed):
    dl = generate_powerlaw(PowerLawSpec(m, n, nnz, seed=seed), DEV)
    _same(dl, synth_oracle.powerlaw(m, n, nnz, seed=seed))
    assert dl.nnz > 0.5 * nnz


@pytest.mark.parametrize("V,E,K,seed", [(40, 300, 7, 0), (200, 3000, 3, 9)])
def test_mcf_bitwise(V, E, K, seed):
    dl = generate_mcf(McfSpec(V, E, K, seed=seed), DEV)
    _same(dl, synth_oracle.mcf(V, E, K, seed=seed))
    assert dl.nnz == 3 * K * E


@pytest.mark.parametrize("kind", ["powerlaw", "mcf"])
def test_generated_lp_solves_like_oracle(kind):
    if kind == "powerlaw":
        p = generate_powerlaw(PowerLawSpec(600, 900, 6000, seed=1), DEV).to_problem()
    else:
        p = generate_mcf(McfSpec(12, 60, 3, seed=1), DEV).to_problem()
    cfg = dict(tolerance=1e-5, seed=1, n_procs=4, grid=(2, 2), max_iterations=40000)
    got = solve(p, SolverConfig(**cfg))
    want = pdhg_oracle.oracle_solve(p, **cfg)
    assert got.status == want.status
    assert (got.iterations, got.restarts) == (want.iterations, want.restarts)
    assert abs(got.objective - want.objective) <= 1e-6 * max(1.0, abs(want.objective))


@pytest.mark.parametrize("m,n,d,seed", [(2000, 3000, 8, 0), (700, 500, 5, 3)])
def test_planted_bitwise(m, n, d, seed):
    from paper_2601_07628_b200.synth import PlantedSpec, generate_planted

    dl = generate_planted(PlantedSpec(m, n, d, seed=seed), DEV)
    want = synth_oracle.planted(m, n, d, seed=seed)
    y = want.pop("y_star")
    _same(dl, want)
    np.testing.assert_array_equal(dl.y_star.cpu().numpy(), y)


def test_planted_optimum_is_reached():
    """The analytic oracle: the solve converges to c·x* (no CPU solve)."""
    from paper_2601_07628_b200.synth import PlantedSpec, generate_planted

    dl = generate_planted(PlantedSpec(3000, 4000, 6, seed=7), DEV)
    star = dl.optimal_objective()
    got = solve(dl.to_problem(), SolverConfig(tolerance=1e-7, seed=7, n_procs=4, grid=(2, 2), max_iterations=200_000))
    assert got.status == "optimal"
    assert abs(got.objective - star) <= 1e-5 * (1.0 + abs(star))


def test_planted_bands_equal_one_piece_instance():
    """Block-by-block generation (small chunks, so the chunk loops run) gives
    the one-piece instance bit for bit: every block, b and c."""
    import scipy.sparse as sp

    from paper_2601_07628_b200.synth import PlantedBands, PlantedSpec

    spec = PlantedSpec(900, 1300, 7, seed=4)
    want = synth_oracle.planted(900, 1300, 7, seed=4)
    A = sp.csr_matrix((want["val"], want["col"], want["ptr"]), shape=(900, 1300))
    bands = PlantedBands(spec, DEV, chunk_draws=7 * 128)
    for (r0, r1), (c0, c1) in (((0, 300), (0, 500)), ((300, 900), (500, 1300)), ((0, 900), (200, 260))):
        blk = bands.block(r0, r1, c0, c1)
        ref = A[r0:r1, c0:c1].tocsr()
        ref.sort_indices()
        np.testing.assert_array_equal(blk.ptr.cpu().numpy(), ref.indptr)
        np.testing.assert_array_equal(blk.col[: blk.nnz].cpu().numpy(), ref.indices)
        np.testing.assert_array_equal(blk.val[: blk.nnz].cpu().numpy(), ref.data)
        lo, hi, y = bands.row_data(r0, r1)
        np.testing.assert_array_equal(lo.cpu().numpy(), want["con_lo"][r0:r1])
        np.testing.assert_array_equal(hi.cpu().numpy(), want["con_hi"][r0:r1])
        c, _, _, x = bands.col_data(c0, c1)
        np.testing.assert_array_equal(c.cpu().numpy(), want["c"][c0:c1])
        np.testing.assert_array_equal(x.cpu().numpy(), want["x_hat"][c0:c1])


def test_band_problem_solves_to_planted_optimum():
    """solve() on a BandProblem: each grid block generated where it lives,
    no global matrix anywhere; reaches the analytic optimum c·x*."""
    from paper_2601_07628_b200.synth import BandProblem, PlantedBands, PlantedSpec, generate_planted

    spec = PlantedSpec(2500, 3500, 6, seed=9)
    star = generate_planted(spec, DEV).optimal_objective()
    prob = BandProblem(PlantedBands(spec, DEV, chunk_draws=6 * 700))
    got = solve(prob, SolverConfig(tolerance=1e-7, seed=9, n_procs=6, grid=(2, 3), permutation="none",
                                   partitioning="uniform", max_iterations=200_000))
    assert got.status == "optimal"
    assert abs(got.objective - star) <= 1e-5 * (1.0 + abs(star))
    assert got.layout["total_nnz"] > 0 and len(got.x) == 3500 and len(got.y) == 2500
    with pytest.raises(ValueError, match="permutation='none'"):
        solve(prob, SolverConfig(n_procs=4, grid=(2, 2)))
