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

from paper_2601_07628_b200 import GridTopology, build_layout  # noqa: E402
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
    a = _solve(p, cfg, engine_overrides={"device_setup": True})
    b = _solve(p, cfg, engine_overrides={"device_setup": False})
    np.testing.assert_array_equal(a.x, b.x)
    np.testing.assert_array_equal(a.y, b.y)
    assert a.layout == b.layout and a.counters == b.counters
