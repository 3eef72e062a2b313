"""Full-size parity at BASELINE cfg2 (1M x 2M, 20M nnz) against the
reference's own solve of the same instance (tests/golden/cfg2_summary.json,
produced by tests/golden/make_golden.py --cfg2 in 713 s of reference CPU time).

Bars: same status / iterations / restarts; objective and the three KKT
residuals within 1e-6 relative (north-star bar); every per-pass log value
within 1e-6 relative. Size-independent properties on top: the generator
reproduces the reference instance (checksums), ⟨Ax, y⟩ = ⟨x, Aᵀy⟩ with the
device products, and a fixed-step trajectory is bit-identical to the CPU
oracle for 8 iterations at full size."""

import json

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2601_07628_b200 import GeneratorSpec, SolverConfig, generate, solve  # noqa: E402


@pytest.fixture(scope="module")
def cfg2():
    return generate(GeneratorSpec(kind="uniform_random", num_rows=1_000_000, num_cols=2_000_000,
                                  nnz_target=20_000_000, inequality_fraction=0.3, seed=0))


@pytest.fixture(scope="module")
def summary():
    return json.loads((GOLDEN / "cfg2_summary.json").read_text())


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def test_instance_matches_reference(cfg2, summary):
    assert float(np.sum(cfg2.con_lower)) == summary["rhs_sum"]
    assert float(np.sum(cfg2.objective)) == summary["c_sum"]
    assert float(np.sum(cfg2.matrix.values)) == summary["vals_sum"]
    nnz = len(cfg2.matrix.col_indices)
    assert int(np.sum(cfg2.matrix.col_indices * (np.arange(nnz) % 1009))) == summary["col_checksum"]


def test_solve_to_1e4_matches_reference(cfg2, summary, caplog):
    import logging

    with caplog.at_level(logging.INFO, logger="gridlp.solver"):
        r = solve(cfg2, SolverConfig(tolerance=1e-4, seed=0))
    exp = summary["result"]
    assert (r.status, r.iterations, r.restarts) == (exp["status"], exp["iterations"], exp["restarts"])
    assert rel(r.objective, exp["objective"]) <= 1e-6
    for k in ("r_primal", "r_dual", "r_gap", "obj_primal", "obj_dual"):
        assert rel(r.report.as_dict()[k], exp["kkt"][k]) <= 1e-6, k
    assert r.counters == exp["counters"]
    assert r.layout == exp["layout"]
    lines = [rec.args for rec in caplog.records if rec.name == "gridlp.solver"]
    assert len(lines) == len(summary["passlog"])
    for got, want in zip(lines, summary["passlog"]):
        assert int(got[0]) == int(want[0]) and int(got[8]) == int(want[8])
        for a, b in zip(got[1:8], want[1:8]):
            assert rel(float(a), b) <= 1e-6 or abs(float(a) - b) <= 1e-12
    assert rel(float(np.sum(r.x)), summary["x_sum"]) <= 1e-9
    np.testing.assert_allclose(r.x[:16], summary["x_head"], rtol=1e-9, atol=1e-12)


def test_adjoint_identity_full_size(cfg2):
    from paper_2601_07628_b200.blocks import DeviceCsr, HostCsr, transpose
    from paper_2601_07628_b200.ops import CudaOps, Fused

    dev = torch.device("cuda", 0)
    A = cfg2.matrix
    h = HostCsr(A.num_rows, A.num_cols, A.row_offsets, A.col_indices, A.values)
    dA, dAT = DeviceCsr(h, dev), DeviceCsr(transpose(h), dev)
    ops = CudaOps(dev, max(dA.slots(), dAT.slots()), 2)
    rng = np.random.default_rng(0)
    x = torch.as_tensor(rng.standard_normal(A.num_cols), device=dev)
    y = torch.as_tensor(rng.standard_normal(A.num_rows), device=dev)
    ax = torch.empty(A.num_rows, dtype=torch.float64, device=dev)
    aty = torch.empty(A.num_cols, dtype=torch.float64, device=dev)
    ops.store(Fused(dA, x), ax)
    ops.store(Fused(dAT, y), aty)
    lhs = float(torch.dot(ax, y))
    rhs = float(torch.dot(x, aty))
    assert abs(lhs - rhs) <= 1e-10 * max(abs(lhs), 1.0)
    import scipy.sparse as sp

    want = sp.csr_matrix((A.values, A.col_indices, A.row_offsets), shape=A.shape).dot(x.cpu().numpy())
    np.testing.assert_array_equal(ax.cpu().numpy(), want)      # all rows <= 45 nnz: bit-exact


def test_fixed_step_trajectory_bitwise_full_size(cfg2):
    from oracle import pdhg_oracle
    from paper_2601_07628_b200 import reference_solve

    class Keep(list):
        keep = {1, 2, 8}

    tr = Keep()
    cfg = dict(tolerance=1e-300, seed=0, eta=0.1, restarts=False, max_iterations=8, power_iterations=1)
    reference_solve(cfg2, SolverConfig(**cfg), trace=tr)
    want = pdhg_oracle.oracle_solve(cfg2, trace_at=[1, 2, 8], **cfg)
    for it, x, y in tr:
        np.testing.assert_array_equal(x, want.trace[it][0])
        np.testing.assert_array_equal(y, want.trace[it][1])
