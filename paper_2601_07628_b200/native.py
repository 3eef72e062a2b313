"""ctypes binding of libgridlp_b200.so (include/gridlp_b200.h) and its build.

The library is the only compute path: if it is missing or no CUDA device is
present, `load()` raises — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, c_double, c_int, c_int32, c_int64, c_uint32, c_void_p
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
LIB_DIR = PKG / "_lib"
LIB_PATH = LIB_DIR / "libgridlp_b200.so"
# the bounds-checked build (-DGRIDLP_CHECKED: every gather index, SELL lane
# extent, long-row range and written row verified in the kernels, a trap on
# violation) — test infrastructure (tests/test_gpu_bounds.py), selected by
# the GRIDLP_LIB environment variable, never by the product path
CHECKED_LIB_PATH = LIB_DIR / "libgridlp_b200_checked.so"
SOURCES = [PKG / "csrc" / "gridlp_b200.cu", PKG / "csrc" / "gridlp_setup.cu", PKG / "csrc" / "gridlp_gen.cu",
           PKG / "csrc" / "gridlp_scale.cu"]
HEADER = ROOT / "include" / "gridlp_b200.h"

MAX_RED = 8
MAX_PARTS = 16
HEAVY_CHUNK = 2048
ROW_MAX_LIMIT = 65536
F_HALPERN = 1
F_SUMSQ = 2
F_STREAM = 4
F_UNIFORM_BOUNDS = 8
CLUSTER_PLAN_LEN = 35

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-std=c++17", "-lineinfo",
    "-Xcompiler", "-fPIC", "-shared",
]


ABI_VERSION = 2
# gridlp_csr_t.val_codec (include/gridlp_b200.h GRIDLP_VALS_*)
VALS_F64, VALS_F32, VALS_UNIT = 0, 1, 2
CSR_WIDE_CTAS = 1   # gridlp_csr_t.launch_flags


LOOP_REC = 12     # GRIDLP_LOOP_REC


class Loop(ctypes.Structure):
    """gridlp_loop_t: the device-side main loop's state (include/gridlp_b200.h)."""
    _fields_ = [("eta", c_double), ("omega", c_double), ("bnorm", c_double), ("cnorm", c_double),
                ("obj_const", c_double), ("tolerance", c_double), ("beta_sufficient", c_double),
                ("beta_necessary", c_double), ("beta_artificial", c_double), ("base_fp", c_double),
                ("prev_fp", c_double), ("total", c_int64), ("inner_k", c_int64), ("max_iterations", c_int64),
                ("kkt_interval", c_int64), ("max_passes", c_int64), ("has_base", c_int32), ("has_prev", c_int32),
                ("restarts", c_int32), ("slot_rows", c_int32), ("slot_cols", c_int32), ("slot_probe", c_int32),
                ("passes", c_int64), ("stopped", c_int32), ("reserved", c_int32)]


class Csr(ctypes.Structure):
    _fields_ = [("num_rows", c_int64), ("num_cols", c_int64), ("nnz", c_int64),
                ("sell_vals", c_void_p), ("sell_cols", c_void_p), ("slice_off", c_void_p),
                ("lane_info", c_void_p), ("num_slices", c_int64),
                ("long_rows", c_void_p), ("long_ptr", c_void_p), ("long_cols", c_void_p),
                ("long_vals", c_void_p), ("num_long_rows", c_int64),
                ("exact_long", c_void_p), ("num_exact_long", c_int64),
                ("chunk_first", c_void_p), ("chunk_row", c_void_p), ("num_chunks", c_int64),
                ("chunk_sums", c_void_p), ("chunk_done", c_void_p),
                ("light_row_max", c_int32), ("exact_row_max", c_int32), ("carry", c_void_p),
                ("hot_cols", c_int64), ("val_codec", c_int32), ("launch_flags", c_int32)]


class Peer(ctypes.Structure):
    _fields_ = [("dst", c_void_p * MAX_PARTS), ("flag", c_void_p * MAX_PARTS), ("recv", c_void_p),
                ("my_flag", c_void_p), ("epoch", c_void_p), ("cta_count", c_void_p), ("group_size", c_int32),
                ("my_slot", c_int32), ("len", c_int64), ("timeout_ns", c_int64)]


class Src(ctypes.Structure):
    _fields_ = [("A", POINTER(Csr)), ("gather", c_void_p),
                ("parts", c_void_p * MAX_PARTS), ("nparts", c_int32),
                ("reserved", c_int32), ("num_rows", c_int64), ("peer", POINTER(Peer))]


class Step(ctypes.Structure):
    _fields_ = [("tau", c_double), ("sigma", c_double), ("gamma", c_double),
                ("inner_k", c_int64)]


class Primal(ctypes.Structure):
    _fields_ = [("x", c_void_p), ("x_bar", c_void_p), ("x_anchor", c_void_p),
                ("c", c_void_p), ("lo", c_void_p), ("hi", c_void_p), ("n", c_int64), ("scale", c_void_p)]


class Dual(ctypes.Structure):
    _fields_ = [("y", c_void_p), ("y_anchor", c_void_p), ("lo", c_void_p),
                ("hi", c_void_p), ("m", c_int64), ("scale", c_void_p)]


TERMS_PER_ROW = 4      # the most reduction terms a fused product op emits per row (KKT columns)


class ClusterKkt(ctypes.Structure):
    _fields_ = [("mode", c_int32), ("reserved", c_int32), ("t_rows", c_void_p), ("t_cols", c_void_p),
                ("t_probe", c_void_p), ("ax", c_void_p), ("xpb", c_void_p)]


class Red(ctypes.Structure):
    _fields_ = [("partials", c_void_p), ("capacity", c_int64), ("out", c_void_p), ("terms", c_void_p),
                ("terms_capacity", c_int64)]


_P = c_void_p
SIGNATURES = {
    "gridlp_abi_version": ([], c_int),
    "gridlp_loop_graph_begin": ([_P, _P], c_int),
    "gridlp_loop_graph_decide": ([_P, _P, _P, _P], c_int),
    "gridlp_loop_graph_end": ([_P, _P], c_int),
    "gridlp_loop_graph_abort": ([_P], c_int),
    "gridlp_build_flags": ([], c_int),
    "gridlp_last_error": ([], ctypes.c_char_p),
    "gridlp_device_info": ([c_int, POINTER(c_int32), POINTER(c_int64)], c_int),
    "gridlp_enable_peer_access": ([c_int], c_int),
    "gridlp_op_slots": ([POINTER(Src)], c_int64),
    "gridlp_set_tuning": ([ctypes.c_char_p, c_int64], c_int),
    "gridlp_get_tuning": ([ctypes.c_char_p], c_int64),
    "gridlp_op_store": ([POINTER(Src), _P, c_uint32, POINTER(Red), _P], c_int),
    "gridlp_op_store_peer": ([POINTER(Src), POINTER(Peer), _P, _P], c_int),
    "gridlp_op_primal": ([POINTER(Src), POINTER(Primal), _P, c_int32, c_uint32, _P], c_int),
    "gridlp_op_dual": ([POINTER(Src), POINTER(Dual), _P, c_int32, c_uint32, _P], c_int),
    "gridlp_op_kkt_rows": ([POINTER(Src), POINTER(Dual), _P, POINTER(Red), _P], c_int),
    "gridlp_op_kkt_cols": ([POINTER(Src), POINTER(Primal), _P, _P, POINTER(Red), _P], c_int),
    "gridlp_op_probe": ([POINTER(Src), POINTER(Dual), _P, _P, _P, POINTER(Red), _P], c_int),
    "gridlp_op_halfdiff_dot": ([_P, _P, _P, c_int64, POINTER(Red), _P], c_int),
    "gridlp_op_anchor": ([_P, _P, c_int64, POINTER(Red), _P], c_int),
    "gridlp_op_dot": ([_P, _P, c_int64, POINTER(Red), _P], c_int),
    "gridlp_op_div": ([_P, _P, c_int64, c_double, _P], c_int),
    "gridlp_op_div_norm": ([_P, _P, c_int64, _P, _P], c_int),
    "gridlp_op_init_primal": ([POINTER(Primal), _P], c_int),
    "gridlp_op_step_advance": ([_P, c_int64, _P], c_int),
    "gridlp_pdhg_iterate": ([POINTER(Src), POINTER(Primal), POINTER(Src), POINTER(Dual), _P, c_int32, c_uint32, _P],
                            c_int),
    "gridlp_iterate_graph_create": ([POINTER(Src), POINTER(Primal), POINTER(Src), POINTER(Dual), _P, c_int32,
                                     c_uint32, POINTER(c_void_p)], c_int),
    "gridlp_graph_launch": ([_P, _P], c_int),
    "gridlp_graph_destroy": ([_P], c_int),
    "gridlp_persistent_scratch_bytes": ([], ctypes.c_size_t),
    "gridlp_cluster_plan": ([POINTER(Src), POINTER(Src), POINTER(c_int64), c_int64], c_int),
    "gridlp_pdhg_iterate_cluster": ([POINTER(Src), POINTER(Primal), POINTER(Src), POINTER(Dual), _P, c_int32,
                                     c_uint32, POINTER(c_int64), POINTER(ClusterKkt), _P], c_int),
    "gridlp_reduce_terms": ([_P, c_int64, c_int32, POINTER(Red), _P], c_int),
    "gridlp_pdhg_iterate_persistent": ([POINTER(Src), POINTER(Primal), POINTER(Src), POINTER(Dual), _P, c_int32,
                                        c_uint32, _P, _P], c_int),
    "gridlp_setup_workspace_bytes": ([c_int64, c_int64], ctypes.c_size_t),
    "gridlp_block_count": ([_P, _P, _P, c_int64, _P, c_int32, c_int32, _P, _P, ctypes.c_size_t, _P], c_int),
    "gridlp_block_fill": ([_P, _P, _P, _P, c_int64, _P, c_int32, c_int32, _P, c_int64, _P, _P, _P,
                           ctypes.c_size_t, _P], c_int),
    "gridlp_csr_transpose": ([_P, _P, _P, c_int64, c_int64, c_int64, _P, _P, _P, _P, ctypes.c_size_t, _P], c_int),
    "gridlp_col_counts": ([_P, c_int64, c_int64, _P, _P], c_int),
    "gridlp_csr_permute": ([_P, _P, _P, c_int64, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P], c_int),
    "gridlp_sell_plan": ([_P, c_int64, c_int32, _P, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P], c_int),
    "gridlp_sell_fill": ([_P, _P, _P, c_int64, c_int32, _P, _P, _P, _P, c_int64, _P, _P, c_int64, _P, _P, _P],
                         c_int),
    "gridlp_gen_workspace_bytes": ([c_int64, c_int64], ctypes.c_size_t),
    "gridlp_gen_scan64": ([_P, _P, c_int64, _P, ctypes.c_size_t, _P], c_int),
    "gridlp_gen_powerlaw_sample": ([ctypes.c_uint64, _P, c_int64, c_int64, c_double, _P, _P], c_int),
    "gridlp_gen_uniform_sample": ([ctypes.c_uint64, _P, c_int64, c_int64, _P, _P], c_int),
    "gridlp_gen_planted_cols": ([ctypes.c_uint64, c_int64, c_int64, c_double, c_double, _P, _P, _P], c_int),
    "gridlp_gen_planted_rows": ([ctypes.c_uint64, c_int64, c_int64, _P, _P, _P, _P, _P], c_int),
    "gridlp_gen_band_draws": ([ctypes.c_uint64, c_int64, c_int64, c_int32, c_int64, _P, _P], c_int),
    "gridlp_gen_planted_row_dot": ([_P, _P, c_int64, c_int64, ctypes.c_uint64, c_double, c_double, _P, _P], c_int),
    "gridlp_gen_col_accumulate": ([_P, _P, _P, c_int64, c_int64, ctypes.c_uint64, _P, _P], c_int),
    "gridlp_gen_add": ([_P, _P, c_int64, _P, _P], c_int),
    "gridlp_gen_sort_rows": ([_P, c_int64, c_int64, _P, _P, _P, ctypes.c_size_t, _P], c_int),
    "gridlp_gen_dedupe_count": ([_P, _P, c_int64, c_int32, c_int32, _P, _P], c_int),
    "gridlp_gen_dedupe_fill": ([_P, _P, c_int64, c_int64, c_int32, c_int32, _P, ctypes.c_uint64, _P, _P, _P], c_int),
    "gridlp_gen_uniform": ([ctypes.c_uint64, ctypes.c_uint64, c_int64, c_int64, c_double, c_double, _P, _P], c_int),
    "gridlp_csr_spmv_seq": ([_P, _P, _P, c_int64, _P, _P, _P], c_int),
    "gridlp_gen_row_bounds": ([ctypes.c_uint64, c_int64, c_double, _P, _P, _P, _P], c_int),
    "gridlp_gen_mcf_row_lengths": ([c_int64, c_int64, c_int64, _P, _P, _P], c_int),
    "gridlp_gen_mcf_fill": ([c_int64, c_int64, c_int64, _P, _P, _P, _P, _P, _P, _P], c_int),
    "gridlp_row_absmax": ([_P, _P, c_int64, _P, _P], c_int),
    "gridlp_row_abssum": ([_P, _P, c_int64, c_int32, _P, _P], c_int),
    "gridlp_col_absmax": ([_P, _P, c_int64, c_int64, _P, _P], c_int),
    "gridlp_update_scale": ([_P, c_int64, _P, _P, _P], c_int),
    "gridlp_scale_matrix": ([_P, _P, _P, c_int64, _P, _P, _P], c_int),
    "gridlp_scale_vector": ([_P, _P, c_int64, c_int32, _P], c_int),
}


def build(verbose: bool = False, force: bool = False, checked: bool = False) -> Path:
    """nvcc the library for sm_100a into the package (in-tree, so it ships
    with the repo snapshot to the GPU box). checked=True builds the
    bounds-checked test variant (CHECKED_LIB_PATH) instead."""
    LIB_DIR.mkdir(exist_ok=True)
    out = CHECKED_LIB_PATH if checked else LIB_PATH
    newest = max(p.stat().st_mtime for p in SOURCES + [HEADER])
    if not force and out.exists() and out.stat().st_mtime >= newest:
        return out
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, *NVCC_FLAGS, "-Xptxas", "-v" if verbose else "-O3", *(["-DGRIDLP_CHECKED"] if checked else []),
           "-I", str(ROOT / "include"), "-o", str(out), *map(str, SOURCES)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stderr[-4000:]}")
    if verbose:
        print(res.stderr)
    return out


class GridlpError(RuntimeError):
    pass


class Library:
    """Loaded libgridlp_b200.so with typed entry points; every call checks
    the returned status and raises GridlpError with gridlp_last_error()."""

    def __init__(self, path: Path = LIB_PATH):
        if not path.exists():
            raise GridlpError(
                f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(no CPU fallback exists)")
        self.path = path
        self._lib = ctypes.CDLL(str(path))
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(self._lib, name)
            fn.argtypes = args
            fn.restype = res
        ver = self._lib.gridlp_abi_version()
        if ver != ABI_VERSION:
            raise GridlpError(f"ABI version {ver} != {ABI_VERSION}")

    def symbols(self):
        return list(SIGNATURES)

    def last_error(self) -> str:
        return self._lib.gridlp_last_error().decode()

    def call(self, name, *args):
        rc = getattr(self._lib, name)(*args)
        if rc != 0:
            raise GridlpError(f"{name} failed ({rc}): {self.last_error()}")
        return rc

    def slots(self, src: Src) -> int:
        return int(self._lib.gridlp_op_slots(ctypes.byref(src)))

    def set_tuning(self, key: str, value: int) -> None:
        """gridlp_set_tuning: kernel choice knobs (bit-identical results)."""
        self.call("gridlp_set_tuning", key.encode(), int(value))

    def get_tuning(self, key: str) -> int:
        return int(self._lib.gridlp_get_tuning(key.encode()))

    def device_info(self, device: int = 0):
        sm = c_int32(0)
        l2 = c_int64(0)
        self.call("gridlp_device_info", device, ctypes.byref(sm), ctypes.byref(l2))
        return sm.value, l2.value


_LIB: Library | None = None


def load() -> Library:
    global _LIB
    if _LIB is None:
        alt = os.environ.get("GRIDLP_LIB")
        _LIB = Library(Path(alt)) if alt else Library()
    return _LIB
