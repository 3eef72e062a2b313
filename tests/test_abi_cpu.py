"""C-ABI library and host-API checks that need no GPU."""

import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2601_07628_b200 import SolverConfig, native

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "gridlp_b200.h").read_text()
    return sorted(set(re.findall(r"^\S.*?\b(gridlp_\w+)\s*\(", text, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    native.build()
    return native.Library()


def test_library_exports_every_header_symbol(lib):
    declared = header_symbols()
    assert declared, "no declarations parsed"
    assert sorted(native.SIGNATURES) == declared
    out = subprocess.run(["nm", "-D", "--defined-only", str(native.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\b(gridlp_\w+)\b", out))
    assert set(declared) <= exported


def test_abi_version_and_error_string(lib):
    assert lib._lib.gridlp_abi_version() == 2
    assert isinstance(lib.last_error(), str)


def test_argument_errors_do_not_touch_the_device(lib):
    # null source -> GRIDLP_ERR_ARG, no launch
    with pytest.raises(native.GridlpError, match="null"):
        lib.call("gridlp_op_store", None, None, 0, None, None)
    bad = native.Csr(4, 4, 2 ** 31, None, None, None, None, 1, 0, 0)
    src = native.Src()
    import ctypes
    src.A = ctypes.pointer(bad)
    with pytest.raises(native.GridlpError, match="2\\^31"):
        lib.call("gridlp_op_store", ctypes.byref(src), 4096, 0, None, None)


def test_sass_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(native.build())], capture_output=True,
                         text=True, check=True).stdout
    assert "sm_100a" in out


def test_config_validation():
    with pytest.raises(ValueError, match="n_procs"):
        SolverConfig(n_procs=2, grid=(2, 2))
    with pytest.raises(ValueError):
        SolverConfig(tolerance=0.0)
    with pytest.raises(ValueError):
        SolverConfig(kkt_interval=0)
    with pytest.raises(ValueError):
        SolverConfig(comm_backend="mpi")
    SolverConfig(comm_backend="threads")  # reference executors alias the device grid
    with pytest.raises(ValueError, match="scaling"):
        SolverConfig(scaling="l2")
    with pytest.raises(ValueError, match="ruiz_iterations"):
        SolverConfig(scaling="ruiz", ruiz_iterations=-1)
    assert SolverConfig().scaling == "none"          # the reference's behaviour by default


def test_solve_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2601_07628_b200 import GeneratorSpec, generate, solve

    p = generate(GeneratorSpec(kind="uniform_random", num_rows=5, num_cols=6, nnz_target=12, seed=0))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        solve(p)


def test_long_row_plan():
    import torch

    from paper_2601_07628_b200.blocks import long_row_plan

    C = native.HEAVY_CHUNK
    lens = np.array([65, 513, C, 4096, 4097, 5 * C - 3, 40 * C])
    hptr = torch.from_numpy(np.concatenate([[0], np.cumsum(lens)]).astype(np.int32))
    exact, first, row = long_row_plan(hptr, 4096)
    np.testing.assert_array_equal(exact.numpy(), np.flatnonzero(lens <= 4096))
    want = np.where(lens > 4096, -(-lens // C), 0)
    np.testing.assert_array_equal(np.diff(first.numpy()), want)
    np.testing.assert_array_equal(row.numpy(), np.repeat(np.arange(len(lens)), want))
    e0, f0, r0 = long_row_plan(torch.zeros(1, dtype=torch.int32), 4096)
    assert f0.tolist() == [0] and r0.numel() == 0 and e0.numel() == 0


def test_sell_layout_roundtrip():
    """The SELL-32 layout holds every light row's entries in their original
    order (lane l of slice s = row 32 s + l), and every long row in the
    compact CSR."""
    from paper_2601_07628_b200.blocks import HostCsr, build_sell

    rng = np.random.default_rng(1)
    m, n = 1300, 900
    lens = rng.integers(0, 50, m)
    lens[[3, 700, 1299]] = [600, 2000, 513]
    lens[10:300] = 0
    ptr = np.concatenate([[0], np.cumsum(lens)])
    col = rng.integers(0, n, int(ptr[-1]))
    val = rng.standard_normal(int(ptr[-1]))
    sd = build_sell(HostCsr(m, n, ptr, col, val), 512)
    assert sd["num_slices"] == -(-m // 32)
    seen = np.zeros(m, dtype=bool)
    off, info = sd["slice_off"], sd["lane_info"]
    for s in range(len(off) - 1):
        for lane in range(32):
            inf = int(info[32 * s + lane])
            if inf < 0:
                continue
            length, local = inf >> 8, inf & 31
            assert local == lane
            row = s * 32 + local
            assert length == lens[row] and not seen[row]
            seen[row] = True
            idx = off[s] + lane + 32 * np.arange(length)
            np.testing.assert_array_equal(sd["cols"][idx], col[ptr[row]:ptr[row + 1]])
            np.testing.assert_array_equal(sd["vals"][idx], val[ptr[row]:ptr[row + 1]])
    heavy = np.flatnonzero(lens > 512)
    np.testing.assert_array_equal(sd["long_rows"], heavy)
    assert np.all(seen == (lens <= 512))
    for h, row in enumerate(heavy):
        a, b = sd["long_ptr"][h], sd["long_ptr"][h + 1]
        np.testing.assert_array_equal(sd["long_cols"][a:b], col[ptr[row]:ptr[row + 1]])


def test_length_order_classes():
    from paper_2601_07628_b200.blocks import length_order

    rng = np.random.default_rng(2)
    lens = rng.integers(0, 100, 5000)
    lens[17] = 10 ** 6
    o = length_order(lens)
    assert sorted(o.tolist()) == list(range(5000)) and o[0] == 17
    cls = np.floor(8 * np.log2(lens[o] + 1.0))
    assert np.all(np.diff(cls) <= 0)                             # longest class first
    ties = np.diff(cls) == 0
    assert np.all(np.diff(o)[ties] > 0)                          # layout order inside a class
    for s in range(0, 4992, 32):                                 # a slice spans <= 2 classes
        ls = lens[o[s:s + 32]]
        if 8 < ls.min() and ls.max() < 1000:
            assert ls.max() <= 1.2 * ls.min() + 1


@pytest.mark.parametrize("K,exact,relabel", [(2, 4096, False), (3, 50, False), (5, 8, False), (3, 4096, True),
                                             (4, 30, True)])
def test_column_band_split(K, exact, relabel):
    """split_column_bands (torch ops, here on CPU tensors): every row's
    entries are distributed over the bands by column range, each band keeps
    the row's entry order, rows longer than exact_row_max go wholly to the
    last band, and concatenating a row's band pieces in band order gives the
    row back (so chaining the bands' sums reproduces the row's add chain)."""
    import torch

    from paper_2601_07628_b200.blocks import DeviceCsrArrays, split_column_bands

    rng = np.random.default_rng(K + exact)
    m, n = 300, 1000
    lens = rng.integers(0, 80, m)
    lens[::9] = 0
    ptr = np.concatenate([[0], np.cumsum(lens)])
    col = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in lens]).astype(np.int32)
    val = rng.standard_normal(len(col))
    # relabel: entries keep ascending LAYOUT columns but are stored under an
    # internal relabeling (the engine's length-class order); to_layout maps back
    to_layout = torch.as_tensor(rng.permutation(n).astype(np.int64)) if relabel else None
    stored = col
    if relabel:
        inv = np.empty(n, np.int64)
        inv[to_layout.numpy()] = np.arange(n)
        stored = inv[col].astype(np.int32)
    arr = DeviceCsrArrays(m, n, len(col), torch.as_tensor(ptr.astype(np.int32)),
                          torch.as_tensor(np.concatenate([stored, np.zeros(8, np.int32)])),
                          torch.as_tensor(np.concatenate([val, np.zeros(8)])))
    cuts = [(k * n) // K for k in range(K + 1)]
    bands = split_column_bands(arr, cuts, exact, to_layout)
    assert len(bands) == K and sum(b.nnz for b in bands) == len(col)
    for r in range(m):
        pieces_c, pieces_v = [], []
        for k, b in enumerate(bands):
            p0, p1 = int(b.ptr[r]), int(b.ptr[r + 1])
            c = b.col[p0:p1].numpy()
            if relabel:
                c = to_layout.numpy()[c]
            if lens[r] > exact:
                assert k == K - 1 or p1 == p0
            elif p1 > p0:
                assert c.min() >= cuts[k] and c.max() < cuts[k + 1]
            pieces_c.append(c)
            pieces_v.append(b.val[p0:p1].numpy())
        np.testing.assert_array_equal(np.concatenate(pieces_c), col[ptr[r]:ptr[r + 1]])
        np.testing.assert_array_equal(np.concatenate(pieces_v), val[ptr[r]:ptr[r + 1]])


def test_tuning_knobs_are_host_only_and_validated(lib):
    """gridlp_set_tuning / gridlp_get_tuning: kernel-choice knobs (no device
    work, so checkable here); unknown keys and out-of-range values are
    GRIDLP_ERR_ARG, get returns -1 for an unknown key."""
    saved = {k: lib.get_tuning(k) for k in ("sell_variant", "chain_products")}
    try:
        lib.set_tuning("sell_variant", 0)
        assert lib.get_tuning("sell_variant") == 0
        lib.set_tuning("chain_products", 0)
        assert lib.get_tuning("chain_products") == 0
        with pytest.raises(native.GridlpError, match="sell_variant"):
            lib.set_tuning("sell_variant", 7)
        with pytest.raises(native.GridlpError, match="unknown key"):
            lib.set_tuning("no_such_knob", 1)
        assert lib.get_tuning("no_such_knob") == -1
    finally:
        for k, v in saved.items():
            lib.set_tuning(k, v)
    assert saved == {"sell_variant": 1, "chain_products": 1}


def test_cluster_and_persistent_entry_points_validate_arguments(lib):
    import ctypes

    with pytest.raises(native.GridlpError, match="bad argument"):
        lib.call("gridlp_pdhg_iterate_persistent", None, None, None, None, None, 1, 0, None, None)
    with pytest.raises(native.GridlpError, match="bad argument"):
        lib.call("gridlp_cluster_plan", None, None, None, 0)
    plan = (ctypes.c_int64 * native.CLUSTER_PLAN_LEN)()
    with pytest.raises(native.GridlpError, match="bad argument"):
        lib.call("gridlp_pdhg_iterate_cluster", None, None, None, None, None, 1, 0, plan, None, None)
    with pytest.raises(native.GridlpError, match="bad argument"):
        lib.call("gridlp_reduce_terms", None, 10, 3, None, None)
    assert int(lib._lib.gridlp_persistent_scratch_bytes()) >= 8
