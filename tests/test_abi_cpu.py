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
    assert lib._lib.gridlp_abi_version() == 1
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


def test_solve_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2601_07628_b200 import GeneratorSpec, generate, solve

    p = generate(GeneratorSpec(kind="uniform_random", num_rows=5, num_cols=6, nnz_target=12, seed=0))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        solve(p)


def test_tile_directory_invariants():
    from paper_2601_07628_b200.blocks import build_tiles

    rng = np.random.default_rng(0)
    lens = rng.integers(0, 40, 5000)
    lens[[7, 100, 4000]] = [3000, 513, 9000]
    lens[200:600] = 0
    ptr = np.concatenate([[0], np.cumsum(lens)])
    t = build_tiles(ptr, 512)
    assert t[0] == 0 and t[-1] == 5000 and np.all(np.diff(t) > 0)
    for a, b in zip(t[:-1], t[1:]):
        nnz = ptr[b] - ptr[a]
        if b - a == 1 and lens[a] > 512:
            continue
        assert b - a <= native.TILE_ROWS
        assert nnz <= native.TILE_NNZ_CAP
        assert np.all(lens[a:b] <= 512)


def test_sell_layout_roundtrip():
    """The SELL-32 window layout (variant 6) holds every light row's entries
    in their original order and every heavy row in the compact CSR."""
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
    assert sd["num_windows"] == -(-m // 256)
    seen = np.zeros(m, dtype=bool)
    off, info = sd["slice_off"], sd["lane_info"]
    for s in range(len(off) - 1):
        for lane in range(32):
            inf = int(info[32 * s + lane])
            if inf < 0:
                continue
            length, local = inf >> 8, inf & 255
            row = (s // 8) * 256 + local
            assert length == lens[row] and not seen[row]
            seen[row] = True
            idx = off[s] + lane + 32 * np.arange(length)
            np.testing.assert_array_equal(sd["cols"][idx], col[ptr[row]:ptr[row + 1]])
            np.testing.assert_array_equal(sd["vals"][idx], val[ptr[row]:ptr[row + 1]])
    heavy = np.flatnonzero(lens > 512)
    np.testing.assert_array_equal(sd["heavy_rows"], heavy)
    assert np.all(seen == (lens <= 512))
    for h, row in enumerate(heavy):
        a, b = sd["heavy_ptr"][h], sd["heavy_ptr"][h + 1]
        np.testing.assert_array_equal(sd["heavy_cols"][a:b], col[ptr[row]:ptr[row + 1]])
