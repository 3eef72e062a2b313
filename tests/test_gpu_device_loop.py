"""The device-side main loop (EngineOptions.device_loop, gridlp_loop_graph_*):
KKT intervals chained on the device by a WHILE-conditional CUDA graph whose
decide kernel evaluates the reference's per-pass logic (pdhg_engine.py:
245-282, :402-476). Bar: a solve with the device loop equals the
host-driven solve BIT FOR BIT — status, iterations, restarts, counters, the
per-pass log (iteration, report, omega, eta, epoch), x and y — on the
cluster path (tiny LP), the kernel-per-product path, with restarts off, an
iteration limit that is not a multiple of the KKT interval, heavy rows, and a
small ring (several launches per epoch); and the golden cfg1 solve still
matches the reference's counts."""

import numpy as np
import pytest
import torch

from conftest import golden_problem

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2601_07628_b200 import GeneratorSpec, LpProblem, SolverConfig, SparseMatrix, generate  # noqa: E402
from paper_2601_07628_b200.api import _solve  # noqa: E402


def _heavy_lp(seed=0, m=700, n=6000):
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, 30, m)
    lens[[3, 100]] = [300, 2000]
    lens[5] = 5000                      # chunked heavy row
    ptr = np.concatenate([[0], np.cumsum(lens)])
    col = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in lens]).astype(np.int64)
    val = rng.standard_normal(len(col))
    x_hat = rng.uniform(1.0, 3.0, n)
    ax = np.array([val[ptr[i]:ptr[i + 1]] @ x_hat[col[ptr[i]:ptr[i + 1]]] for i in range(m)])
    return LpProblem(SparseMatrix(m, n, ptr, col, val), rng.standard_normal(n), np.zeros(n), np.full(n, 4.0),
                     ax - 0.5, ax + 0.5)


def _run(p, cfg, **over):
    log = []

    class Hook:
        pass

    from paper_2601_07628_b200 import engine as eng

    orig = eng.PdhgEngine.run

    def run(self, eta, omega, trace=None, log_hook=None):
        def hook(total, report, omega_, eta_, epoch):
            log.append((total, report.r_primal, report.r_dual, report.r_gap, report.obj_primal, omega_, eta_,
                        epoch))
            if log_hook is not None:
                log_hook(total, report, omega_, eta_, epoch)
        return orig(self, eta, omega, trace, hook)

    eng.PdhgEngine.run = run
    try:
        r = _solve(p, SolverConfig(**cfg), engine_overrides=over)
    finally:
        eng.PdhgEngine.run = orig
    return r, log


def _same(a, b):
    (ra, la), (rb, lb) = a, b
    assert (ra.status, ra.iterations, ra.restarts) == (rb.status, rb.iterations, rb.restarts)
    assert ra.counters == rb.counters
    assert ra.objective == rb.objective
    np.testing.assert_array_equal(ra.x, rb.x)
    np.testing.assert_array_equal(ra.y, rb.y)
    assert la == lb and len(la) > 0


CASES = {
    "cluster": (lambda: generate(GeneratorSpec(kind="uniform_random", num_rows=600, num_cols=1000, nnz_target=6000,
                                               inequality_fraction=0.3, seed=2)),
                dict(tolerance=1e-6, seed=2), {}),
    "products": (lambda: generate(GeneratorSpec(kind="uniform_random", num_rows=600, num_cols=1000,
                                                nnz_target=6000, inequality_fraction=0.3, seed=2)),
                 dict(tolerance=1e-6, seed=2), {"cluster_small": False}),
    "heavy": (_heavy_lp, dict(tolerance=1e-6, seed=1, max_iterations=5000), {}),
    "no_restarts_limit": (_heavy_lp, dict(tolerance=1e-9, seed=1, restarts=False, max_iterations=1000), {}),
    "small_ring": (lambda: generate(GeneratorSpec(kind="uniform_random", num_rows=400, num_cols=700,
                                                  nnz_target=3000, inequality_fraction=0.3, seed=4)),
                   dict(tolerance=1e-6, seed=4), {"device_loop_passes": 3}),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_device_loop_equals_host_loop(name):
    make, cfg, over = CASES[name]
    p = make()
    dev = _run(p, cfg, device_loop=True, **over)
    host = _run(p, cfg, device_loop=False, **over)
    _same(dev, host)


def test_device_loop_golden_cfg1(golden_cfg1):
    z = golden_cfg1
    for over in ({}, {"cluster_small": False}):
        r, log = _run(golden_problem(z), dict(tolerance=1e-4, seed=0), device_loop=True, **over)
        assert (r.status, r.iterations, r.restarts) == ("optimal", int(z["iterations"]), int(z["restarts"]))
        assert abs(r.objective - float(z["result_objective"])) <= 1e-6 * abs(float(z["result_objective"]))
        assert len(log) == int(z["iterations"]) // 64
