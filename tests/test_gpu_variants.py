"""Every light-row kernel variant (gridlp_set_tuning "sell_variant") and the
chained products of gridlp_pdhg_iterate ("chain_products") compute the same
bits: the knobs pick kernels, never arithmetic. Products vs scipy's
csr_matvec (the reference kernel, sparse_kernels.py:18-24) bit for bit on
rows <= 4096 entries, reductions vs the default variant bit for bit, and a
fixed-step restart-free trajectory identical across variants and to the CPU
oracle (pdhg_engine.py:223-242)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import pdhg_oracle  # noqa: E402
from paper_2601_07628_b200 import GeneratorSpec, SolverConfig, generate, native, reference_solve  # noqa: E402
from paper_2601_07628_b200.blocks import DeviceCsr, HostCsr  # noqa: E402
from paper_2601_07628_b200.ops import CudaOps, Fused  # noqa: E402

DEV = torch.device("cuda", 0)
VARIANTS = [0, 1]


@pytest.fixture
def tuning():
    lib = native.load()
    keys = ("sell_variant", "chain_products", "wide_ctas")
    saved = {k: lib.get_tuning(k) for k in keys}
    yield lib
    for k, v in saved.items():
        lib.set_tuning(k, v)


def _matrix(seed, m=4000, n=6000):
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, 90, m)
    lens[rng.choice(m, 40, replace=False)] = rng.integers(129, 3000, 40)     # long rows
    lens[11] = 6000                                                          # heavy (> 4096)
    lens[200:260] = 0
    ptr = np.concatenate([[0], np.cumsum(lens)])
    col = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in lens]).astype(np.int64)
    val = rng.standard_normal(len(col)) * 10.0 ** rng.integers(-5, 5, len(col))
    return HostCsr(m, n, ptr, col, val), lens


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("light", [128, 1024])
def test_products_bitwise_every_variant(tuning, variant, light):
    import scipy.sparse as sp

    tuning.set_tuning("sell_variant", variant)
    h, lens = _matrix(variant + 7 * light)
    rng = np.random.default_rng(1)
    x = rng.standard_normal(h.num_cols)
    want = sp.csr_matrix((h.val, h.col, h.ptr), shape=(h.num_rows, h.num_cols)).dot(x)
    A = DeviceCsr(h, DEV, light_row_max=light)
    ops = CudaOps(DEV, A.slots() + 8, 4)
    ops.enable_terms(h.num_rows)               # canonical (layout-independent) reductions, as the engine
    out = torch.full((h.num_rows,), np.nan, dtype=torch.float64, device=DEV)
    xd = torch.as_tensor(x, device=DEV)
    ops.store(Fused(A, xd), out, slot=0)       # + fused sum of squares
    got = out.cpu().numpy()
    exact = lens <= 4096
    np.testing.assert_array_equal(got[exact], want[exact])
    assert np.max(np.abs(got[~exact] - want[~exact])) <= 1e-12 * np.abs(want[~exact]).max()
    sq = float(ops.read_slots(1)[0, 0])
    tuning.set_tuning("sell_variant", 0)
    ops0 = CudaOps(DEV, A.slots() + 8, 4)
    ops0.enable_terms(h.num_rows)
    out0 = torch.empty_like(out)
    ops0.store(Fused(A, xd), out0, slot=0)
    assert torch.equal(out, out0)
    assert sq == float(ops0.read_slots(1)[0, 0])     # canonical row-order reduction
    A.struct.hot_cols = h.num_cols // 3              # reserved field: ignored by the kernels
    out1 = torch.empty_like(out)
    ops0.store(Fused(A, xd), out1)
    assert torch.equal(out, out1)


@pytest.mark.parametrize("variant,chain", [(0, 0), (0, 1), (1, 1), (1, 0)])
def test_fixed_step_trajectory_every_variant(tuning, variant, chain):
    tuning.set_tuning("sell_variant", variant)
    tuning.set_tuning("chain_products", chain)
    p = generate(GeneratorSpec(kind="uniform_random", num_rows=3000, num_cols=5000, nnz_target=60000,
                               inequality_fraction=0.3, seed=4))

    class Keep(list):
        keep = {1, 37, 200}

    cfg = dict(tolerance=1e-300, seed=0, eta=0.05, restarts=False, max_iterations=200, power_iterations=3)
    tr = Keep()
    got = reference_solve(p, SolverConfig(**cfg), trace=tr)
    want = pdhg_oracle.oracle_solve(p, trace_at=[1, 37, 200], **cfg)
    for it, x, y in tr:
        np.testing.assert_array_equal(x, want.trace[it][0])
        np.testing.assert_array_equal(y, want.trace[it][1])
    # and through the captured-graph main loop (no trace): final iterate
    r = reference_solve(p, SolverConfig(**cfg))
    np.testing.assert_array_equal(r.x, want.x)
    assert got.iterations == r.iterations == 200


@pytest.mark.parametrize("heavy", [False, True])
def test_persistent_launch_equals_graph_path(heavy):
    """gridlp_pdhg_iterate_persistent (one cooperative launch per chunk, grid
    barriers between the products) reproduces the kernel-per-product path bit
    for bit, with long exact rows (warp per row); heavy rows fall back."""
    from paper_2601_07628_b200.api import _solve
    from paper_2601_07628_b200.problem import LpProblem, SparseMatrix

    rng = np.random.default_rng(5)
    m, n = 900, 7000
    lens = rng.integers(1, 40, m)
    lens[[2, 50, 400]] = [300, 1500, 4000]
    if heavy:
        lens[7] = 6000
    ptr = np.concatenate([[0], np.cumsum(lens)])
    col = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in lens]).astype(np.int64)
    val = rng.standard_normal(len(col))
    xh = rng.uniform(1, 3, n)
    ax = np.array([val[ptr[i]:ptr[i + 1]] @ xh[col[ptr[i]:ptr[i + 1]]] for i in range(m)])
    p = LpProblem(SparseMatrix(m, n, ptr, col, val), rng.standard_normal(n), np.zeros(n), np.full(n, 4.0),
                  ax - 0.3, ax + 0.3)
    cfg = SolverConfig(tolerance=1e-7, seed=3, max_iterations=3000)
    a = _solve(p, cfg, engine_overrides={"persistent_max_nnz": 1 << 30})
    b = _solve(p, cfg, engine_overrides={"persistent_max_nnz": 0})
    assert (a.status, a.iterations, a.restarts) == (b.status, b.iterations, b.restarts)
    np.testing.assert_array_equal(a.x, b.x)
    np.testing.assert_array_equal(a.y, b.y)
    assert a.report == b.report


@pytest.mark.parametrize("seed", [0, 1])
def test_cluster_launch_equals_graph_path(seed):
    """gridlp_pdhg_iterate_cluster (one 8-CTA cluster launch per chunk:
    replicated vectors and the matrix in shared memory, DSMEM broadcasts,
    cluster barriers) reproduces the kernel-per-product path bit for bit on
    BASELINE cfg1-shaped LPs; an LP with long rows falls back by itself."""
    from paper_2601_07628_b200.api import _solve

    p = generate(GeneratorSpec(kind="uniform_random", num_rows=2000, num_cols=4000, nnz_target=20000,
                               inequality_fraction=0.3, seed=seed))
    cfg = SolverConfig(tolerance=1e-6, seed=seed, max_iterations=4000)
    a = _solve(p, cfg, engine_overrides={"cluster_small": True})
    b = _solve(p, cfg, engine_overrides={"cluster_small": False})
    assert (a.status, a.iterations, a.restarts) == (b.status, b.iterations, b.restarts)
    np.testing.assert_array_equal(a.x, b.x)
    np.testing.assert_array_equal(a.y, b.y)
    assert a.report == b.report


@pytest.mark.parametrize("light", [128, 1024])
def test_wide_cta_launch_hint_bitwise(tuning, light):
    """GRIDLP_CSR_WIDE_CTAS (4-warp CTAs for the SELL lanes of main-loop /
    store products) computes the same rows bit for bit, including a slice
    count that is not a multiple of 4; the engine sets it for blocks of very
    short rows only (blocks.WIDE_CTA_MAX_MEAN_ROW)."""
    from paper_2601_07628_b200.blocks import WIDE_CTA_MAX_MEAN_ROW

    h, lens = _matrix(11 + light)
    x = torch.as_tensor(np.random.default_rng(3).standard_normal(h.num_cols), device=DEV)
    A = DeviceCsr(h, DEV, light_row_max=light)
    assert (A.struct.launch_flags & native.CSR_WIDE_CTAS) == 0       # mean row length > 6
    ops = CudaOps(DEV, A.slots() + 8, 4)
    want = torch.empty(h.num_rows, dtype=torch.float64, device=DEV)
    ops.store(Fused(A, x), want)
    A.struct.launch_flags |= native.CSR_WIDE_CTAS
    got = torch.full_like(want, np.nan)
    ops.store(Fused(A, x), got)
    assert torch.equal(got, want)
    tuning.set_tuning("wide_ctas", 0)
    off = torch.full_like(want, np.nan)
    ops.store(Fused(A, x), off)
    assert torch.equal(off, want)
    tuning.set_tuning("wide_ctas", 1)
    # a block of 3-entry rows (an MCF column's shape) gets the hint
    m, n = 1000, 700
    ptr = np.arange(0, 3 * m + 1, 3)
    col = np.sort(np.random.default_rng(5).integers(0, n, (m, 3)), axis=1).ravel()
    col[1::3] = np.minimum(col[1::3] + 1, n - 1)
    short = DeviceCsr(HostCsr(m, n, ptr, col.astype(np.int64), np.ones(3 * m)), DEV)
    assert 3.0 <= WIDE_CTA_MAX_MEAN_ROW and short.struct.launch_flags & native.CSR_WIDE_CTAS
