"""Compact value codecs (gridlp_csr_t.val_codec, include/gridlp_b200.h
GRIDLP_VALS_*): a block whose values are all +-1 (network / multi-commodity
flow rows) or all exact floats (small integer coefficients) is stored with
4 resp. 8 bytes per nonzero instead of 12. The kernels rebuild the exact
FP64 value before the same multiply, so the bar is BIT-IDENTICAL products —
light, long-exact and chunked heavy rows, every light-row kernel variant —
and bit-identical solves (reference: the sequential scipy csr_matvec of
sparse_kernels.py:18-24, on the FP64 values of lp_model.py:53-55)."""

import numpy as np
import pytest
import torch

from oracle import pdhg_oracle

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2601_07628_b200 import SolverConfig, native  # noqa: E402
from paper_2601_07628_b200.api import _solve  # noqa: E402
from paper_2601_07628_b200.blocks import DeviceCsr, HostCsr  # noqa: E402
from paper_2601_07628_b200.ops import CudaOps, Fused  # noqa: E402

DEV = torch.device("cuda", 0)


@pytest.fixture(scope="module")
def ops():
    return CudaOps(DEV, 1 << 16, 16)


def _matrix(kind, seed):
    rng = np.random.default_rng(seed)
    m, n = 2500, 9000
    lens = rng.integers(0, 40, m)
    lens[[3, 400, 1500]] = [700, 3000, 4096]         # long exact rows
    lens[[9, 2000]] = [6000, 2 * native.HEAVY_CHUNK + 17]   # heavy (chunked) rows
    lens[50:90] = 0
    ptr = np.concatenate([[0], np.cumsum(lens)])
    col = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in lens]).astype(np.int64)
    k = len(col)
    if kind == "unit":
        val = rng.choice([-1.0, 1.0], k)
    elif kind == "int":
        val = rng.integers(-300, 300, k).astype(np.float64)
        val[val == 0] = 7.0
    elif kind == "half":                              # dyadic, exact in float32, incl. -0.0 and inf
        val = rng.integers(-4096, 4096, k) / 64.0
        val[::97] = -0.0
        val[5] = np.inf
    else:
        val = rng.standard_normal(k)
    x = rng.standard_normal(n)
    x[[0, 17, 4000]] = [np.nan, np.inf, -0.0]
    return HostCsr(m, n, ptr, col, val), x


@pytest.mark.parametrize("variant", [1, 0])
@pytest.mark.parametrize("kind,codecs,auto", [("unit", ("unit", "f32"), "unit"), ("int", ("f32",), "f32"),
                                              ("half", ("f32",), "f32"), ("normal", (), "f64")])
def test_products_bitwise(ops, kind, codecs, auto, variant):
    lib = native.load()
    old = lib.get_tuning("sell_variant")
    lib.set_tuning("sell_variant", variant)
    try:
        for seed in range(2):
            h, x = _matrix(kind, seed)
            xd = torch.as_tensor(x, device=DEV)
            ref = DeviceCsr(h, DEV, light_row_max=128)
            assert ref.codec == "f64" and ref.heavy_rows == 2
            want = torch.empty(h.num_rows, dtype=torch.float64, device=DEV)
            ops.store(Fused(ref, xd), want)
            a = DeviceCsr(h, DEV, light_row_max=128, value_codec="auto")
            assert a.codec == auto
            for c in codecs + ("auto",):
                A = DeviceCsr(h, DEV, light_row_max=128, value_codec=c)
                got = torch.full_like(want, 12345.0)
                ops.store(Fused(A, xd), got)
                np.testing.assert_array_equal(got.cpu().numpy(), want.cpu().numpy(), err_msg=f"{kind}/{c}")
                if A.val_codec == native.VALS_UNIT:
                    assert A.dev["vals"].numel() == 0 and A.dev["long_vals"].numel() == 0
                    assert A.bytes_per_product() == ref.bytes_per_product() - 8 * h.nnz
    finally:
        lib.set_tuning("sell_variant", old)


def test_forced_codec_must_be_lossless():
    h, _ = _matrix("normal", 0)
    with pytest.raises(ValueError, match="not lossless"):
        DeviceCsr(h, DEV, value_codec="f32")
    h, _ = _matrix("int", 0)
    with pytest.raises(ValueError, match="not lossless"):
        DeviceCsr(h, DEV, value_codec="unit")
    with pytest.raises(ValueError, match="value_codec"):
        DeviceCsr(h, DEV, value_codec="bf16")


def test_fused_epilogue_and_reductions_bitwise(ops):
    """A fused reduction (sum of squares of the product, the power
    iteration's op) over a UNIT block equals the FP64 block's bit for bit."""
    h, x = _matrix("unit", 3)
    x = np.nan_to_num(x, nan=0.5, posinf=2.0)
    xd = torch.as_tensor(x, device=DEV)
    outs, ssq = [], []
    for c in ("f64", "unit"):
        A = DeviceCsr(h, DEV, value_codec=c)
        out = torch.empty(h.num_rows, dtype=torch.float64, device=DEV)
        ops.store(Fused(A, xd), out, slot=0)
        ssq.append(float(ops.read_slots(1)[0][0]))
        outs.append(out.cpu().numpy())
    np.testing.assert_array_equal(outs[0], outs[1])
    assert ssq[0] == ssq[1]


@pytest.mark.parametrize("grid", [(1, 1), (2, 2)])
def test_mcf_solve_identical_with_unit_codec(grid):
    """Generated multi-commodity flow LP (every value +-1): the solve with
    the UNIT codec forced on every block equals the FP64-stored solve bit
    for bit (x, y, iterations, restarts, objective) and the CPU oracle's
    status / counts / objective."""
    from paper_2601_07628_b200.synth import McfSpec, generate_mcf

    p = generate_mcf(McfSpec(30, 200, 4, seed=2), DEV).to_problem()
    cfg = dict(tolerance=1e-5, seed=1, n_procs=grid[0] * grid[1], grid=grid, max_iterations=30000)
    res = {}
    for c in ("f64", "auto"):
        over = dict(value_codec=c, value_codec_min_nnz=0, cluster_small=False)
        res[c] = _solve(p, SolverConfig(**cfg), engine_overrides=over)
    a, b = res["f64"], res["auto"]
    assert (a.status, a.iterations, a.restarts) == (b.status, b.iterations, b.restarts)
    assert a.objective == b.objective
    np.testing.assert_array_equal(a.x, b.x)
    np.testing.assert_array_equal(a.y, b.y)
    want = pdhg_oracle.oracle_solve(p, **cfg)
    assert (b.status, b.iterations, b.restarts) == (want.status, want.iterations, want.restarts)
    assert abs(b.objective - want.objective) <= 1e-6 * max(1.0, abs(want.objective))


def test_engine_records_codec_choice():
    """The engine picks UNIT for the MCF blocks (both orientations) above
    value_codec_min_nnz and FP64 below it."""
    from paper_2601_07628_b200.api import prepare
    from paper_2601_07628_b200.synth import McfSpec, generate_mcf

    p = generate_mcf(McfSpec(30, 200, 4, seed=2), DEV).to_problem()
    cfg = SolverConfig(tolerance=1e-5, seed=1)
    eng = prepare(p, cfg, device=DEV, engine_overrides=dict(value_codec_min_nnz=0))[0]
    assert set(eng.choices["value_codec"].values()) == {"unit"}
    eng = prepare(p, cfg, device=DEV)[0]
    assert set(eng.choices["value_codec"].values()) == {"f64"}     # 2400 nnz < the 1M default
