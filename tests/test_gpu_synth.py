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
