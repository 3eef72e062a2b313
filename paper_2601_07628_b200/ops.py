"""Device operations of the engine, bound to libgridlp_b200.so.

`CudaOps` is the only implementation in the package: each method is one
C-ABI call (include/gridlp_b200.h) on the current CUDA stream. ctypes
argument structs are built once per engine object and cached, so a
captured chunk of iterations is a plain sequence of kernel launches.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import native
from .blocks import BandedCsr, DeviceCsr, parts_src


class Fused:
    """Sums come from a product of one local block with a gather vector."""

    def __init__(self, mat: DeviceCsr, gather: torch.Tensor):
        self.mat = mat
        self.gather = gather
        self.num_rows = mat.num_rows


class Parts:
    """Sums come from an ascending-order sum of partial vectors."""

    def __init__(self, parts, num_rows: int):
        self.parts = list(parts)
        self.num_rows = int(num_rows)


class PeerDest:
    """Destination of a product in a peer exchange (comm.PeerAxis), with an
    optional local copy of the partial."""

    def __init__(self, axis, local=None):
        self.axis = axis
        self.local = local


class PeerSrc:
    """Sums are the G slots of a peer exchange (comm.PeerAxis), in order."""

    def __init__(self, axis, num_rows: int):
        self.axis = axis
        self.num_rows = int(num_rows)


def _heavy(src) -> int:
    """Extra kernels a product launches for its long rows (warp-per-row and
    heavy-chunk kernels, when present)."""
    return src.mat.launches() - 1 if isinstance(src, Fused) else 0


def _pflags(col, halpern: bool) -> int:
    """Flags of a primal op: Halpern, and uniform variable bounds (the op
    then reads lo[0], hi[0] instead of two n-vectors)."""
    return (native.F_HALPERN if halpern else 0) | (native.F_UNIFORM_BOUNDS if getattr(col, "uniform_bounds", False)
                                                   else 0)


def _ptr(t):
    return t.data_ptr() if t is not None and t.numel() else None


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None) or (
    lambda idx: torch.cuda.current_stream(idx).cuda_stream)


class _IterateGraph:
    """A captured chunk of iterations (gridlp_iterate_graph_create)."""

    def __init__(self, ops, handle, launches: int):
        self.ops, self.handle, self.launches = ops, handle, launches

    def replay(self):
        self.ops.lib.call("gridlp_graph_launch", self.handle, self.ops.stream())
        self.ops.launches += self.launches

    def __del__(self):
        try:
            if self.handle:
                self.ops.lib._lib.gridlp_graph_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


class CudaOps:
    kind = "cuda"

    def __init__(self, device: torch.device, capacity: int, num_slots: int):
        self.lib = native.load()
        self.device = device
        self._dev_index = torch.device(device).index if torch.device(device).index is not None else (
            torch.cuda.current_device() if torch.cuda.is_available() else 0)
        self.capacity = max(int(capacity), 1)
        self.partials = torch.zeros(self.capacity * native.MAX_RED, dtype=torch.float64, device=device)
        self.slots = torch.zeros((max(num_slots, 1), native.MAX_RED), dtype=torch.float64, device=device)
        self.slots_host = torch.zeros_like(self.slots, device="cpu").pin_memory()
        self.step = torch.zeros(4, dtype=torch.float64, device=device)
        self.step_host = torch.zeros(4, dtype=torch.float64).pin_memory()
        self._red = {}
        self._srcs = {}
        self.launches = 0          # kernels launched through this object

    # -- plumbing ------------------------------------------------------------
    def stream(self):
        # the current stream's raw handle (inside a torch graph capture: the
        # capture stream); the raw query costs well under a microsecond where
        # torch.cuda.current_stream() builds a Stream object (~7 µs a call,
        # ~10 calls per KKT pass)
        return _raw_stream(self._dev_index)

    def enable_terms(self, rows: int):
        """Canonical (layout-independent) reductions for fused products of up
        to `rows` rows: a per-row term buffer (gridlp_red_t.terms)."""
        self.terms = torch.empty(max(int(rows), 1) * native.TERMS_PER_ROW, dtype=torch.float64, device=self.device)
        self._red = {}

    def red(self, slot: int):
        r = self._red.get(slot)
        if r is None:
            t = getattr(self, "terms", None)
            r = native.Red(self.partials.data_ptr(), self.capacity, self.slots[slot].data_ptr(),
                           t.data_ptr() if t is not None else None, t.numel() if t is not None else 0)
            self._red[slot] = r
        return ctypes.byref(r)

    def src(self, s):
        key = id(s)
        hit = self._srcs.get(key)
        if isinstance(s, Fused) and isinstance(s.mat, BandedCsr):
            # leading column bands: running row sums into the block's carry
            # buffer (launched on every use, so graphs capture them too)
            key2 = ("bands", key)
            hit2 = self._srcs.get(key2)
            if hit2 is None or hit2[0] is not s:
                hit2 = (s, [b.src(s.gather) for b in s.mat.bands[:-1]])
                self._srcs[key2] = hit2
            for c in hit2[1]:
                self.lib.call("gridlp_op_store", ctypes.byref(c), s.mat.acc.data_ptr(), native.F_STREAM, None,
                              self.stream())
        if hit is not None and hit[0] is s:
            return ctypes.byref(hit[1])
        if isinstance(s, Fused):
            c = s.mat.src(s.gather)
        elif isinstance(s, PeerSrc):
            c = parts_src([], s.num_rows)
            c.peer = ctypes.pointer(s.axis.struct)
        else:
            c = parts_src(s.parts, s.num_rows)
        self._srcs[key] = (s, c)
        return ctypes.byref(c)

    @staticmethod
    def primal_struct(col):
        c = getattr(col, "_cprimal", None)
        if c is None:
            c = native.Primal(_ptr(col.x), _ptr(col.xbar), _ptr(col.x0), _ptr(col.c),
                              _ptr(col.lo), _ptr(col.hi), col.n, _ptr(getattr(col, "scale", None)))
            col._cprimal = c
        return ctypes.byref(c)

    @staticmethod
    def dual_struct(row):
        c = getattr(row, "_cdual", None)
        if c is None:
            c = native.Dual(_ptr(row.y), _ptr(row.y0), _ptr(row.lo), _ptr(row.hi), row.m,
                            _ptr(getattr(row, "scale", None)))
            row._cdual = c
        return ctypes.byref(c)

    def set_step(self, tau: float, sigma: float, gamma: float, inner_k: int):
        # the pinned staging buffer may still be read by the previous async
        # copy (e.g. finish() right after a partial chunk): wait for it first
        ev = getattr(self, "_step_ev", None)
        if ev is not None:
            ev.synchronize()
        h = self.step_host
        h[0], h[1], h[2] = tau, sigma, gamma
        h.view(torch.int64)[3] = int(inner_k)
        self.step.copy_(h, non_blocking=True)
        if ev is None:
            ev = self._step_ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))

    def read_slots(self, n: int) -> np.ndarray:
        self.slots_host[:n].copy_(self.slots[:n], non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        return self.slots_host[:n].numpy().copy()

    # -- ops -----------------------------------------------------------------
    def store(self, src, out, slot=None):
        if isinstance(out, PeerDest):
            self.launches += 1 + _heavy(src)
            self.lib.call("gridlp_op_store_peer", self.src(src), ctypes.byref(out.axis.struct), _ptr(out.local),
                          self.stream())
            return
        self.launches += (2 if slot is not None else 1) + _heavy(src)
        flags = native.F_SUMSQ if slot is not None else 0
        self.lib.call("gridlp_op_store", self.src(src), _ptr(out), flags,
                      self.red(slot) if slot is not None else None, self.stream())

    def primal(self, src, col, it: int, halpern: bool):
        self.launches += 1 + _heavy(src)
        self.lib.call("gridlp_op_primal", self.src(src), self.primal_struct(col),
                      self.step.data_ptr(), it, _pflags(col, halpern), self.stream())

    def dual(self, src, row, it: int, halpern: bool):
        self.launches += 1 + _heavy(src)
        self.lib.call("gridlp_op_dual", self.src(src), self.dual_struct(row),
                      self.step.data_ptr(), it, native.F_HALPERN if halpern else 0, self.stream())

    def kkt_rows(self, src, row, ax, slot):
        self.launches += 2 + _heavy(src)
        self.lib.call("gridlp_op_kkt_rows", self.src(src), self.dual_struct(row), _ptr(ax),
                      self.red(slot), self.stream())

    def kkt_cols(self, src, col, slot):
        self.launches += 2 + _heavy(src)
        self.lib.call("gridlp_op_kkt_cols", self.src(src), self.primal_struct(col), _ptr(col.xpb),
                      self.step.data_ptr(), self.red(slot), self.stream())

    def probe(self, src, row, ax, dy_out, slot):
        self.launches += 2 + _heavy(src)
        self.lib.call("gridlp_op_probe", self.src(src), self.dual_struct(row), _ptr(ax), _ptr(dy_out),
                      self.step.data_ptr(), self.red(slot), self.stream())

    def halfdiff_dot(self, a, b, d, slot):
        self.launches += 2
        self.lib.call("gridlp_op_halfdiff_dot", _ptr(a), _ptr(b), _ptr(d), a.numel(),
                      self.red(slot), self.stream())

    def anchor(self, v, anchor, slot):
        self.launches += 2
        self.lib.call("gridlp_op_anchor", _ptr(v), _ptr(anchor), v.numel(), self.red(slot), self.stream())

    def dot(self, a, b, slot):
        self.launches += 2
        self.lib.call("gridlp_op_dot", _ptr(a), _ptr(b), a.numel(), self.red(slot), self.stream())

    def div(self, inp, out, divisor: float):
        self.launches += 1
        self.lib.call("gridlp_op_div", _ptr(inp), _ptr(out), inp.numel(), float(divisor), self.stream())

    def div_norm(self, inp, out, slot: int):
        self.launches += 1
        self.lib.call("gridlp_op_div_norm", _ptr(inp), _ptr(out), inp.numel(), self.slots[slot].data_ptr(),
                      self.stream())

    def init_primal(self, col):
        self.launches += 1
        self.lib.call("gridlp_op_init_primal", self.primal_struct(col), self.stream())

    def iterate(self, psrc, col, dsrc, row, count: int, halpern: bool):
        """count fused iterations of a single-block grid in one C call
        (gridlp_pdhg_iterate), step counter advanced on the device."""
        self.launches += count * (2 + _heavy(psrc) + _heavy(dsrc)) + (1 if count else 0)
        self.lib.call("gridlp_pdhg_iterate", self.src(psrc), self.primal_struct(col), self.src(dsrc),
                      self.dual_struct(row), self.step.data_ptr(), int(count), _pflags(col, halpern),
                      self.stream())

    def iterate_persistent(self, psrc, col, dsrc, row, count: int, halpern: bool) -> bool:
        """count fused iterations of a single-block grid in one cooperative
        launch (gridlp_pdhg_iterate_persistent). False (nothing launched)
        when the blocks have heavy rows: the caller uses iterate()."""
        scratch = getattr(self, "_persist_scratch", None)
        if scratch is None:
            nbytes = int(self.lib._lib.gridlp_persistent_scratch_bytes())
            scratch = self._persist_scratch = torch.zeros(max(nbytes // 8, 1), dtype=torch.float64,
                                                          device=self.device)
        rc = self.lib._lib.gridlp_pdhg_iterate_persistent(
            self.src(psrc), self.primal_struct(col), self.src(dsrc), self.dual_struct(row), self.step.data_ptr(),
            int(count), native.F_HALPERN if halpern else 0, scratch.data_ptr(), self.stream())
        if rc == 4:              # GRIDLP_ERR_UNSUPPORTED
            return False
        if rc != 0:
            raise native.GridlpError(f"gridlp_pdhg_iterate_persistent failed ({rc}): {self.lib.last_error()}")
        self.launches += 1 if count else 0
        return True

    def iterate_graph(self, psrc, col, dsrc, row, count: int, halpern: bool):
        """A chunk of `count` fused iterations of a single-block grid
        captured once in C (gridlp_iterate_graph_create) — no torch capture
        machinery, no synchronisation; replay with graph_launch()."""
        h = ctypes.c_void_p()
        self.lib.call("gridlp_iterate_graph_create", self.src(psrc), self.primal_struct(col), self.src(dsrc),
                      self.dual_struct(row), self.step.data_ptr(), int(count), _pflags(col, halpern), ctypes.byref(h))
        launches = count * (2 + _heavy(psrc) + _heavy(dsrc)) + 1
        return _IterateGraph(self, h, launches)

    def loop_graph(self, build, loop_dev: torch.Tensor, ring_dev: torch.Tensor):
        """The device-side main loop (gridlp_loop_graph_*): build() issues one
        KKT interval's launches on this ops' current stream while it is
        captured into the body of a WHILE-conditional graph, followed by the
        decide kernel over this ops' reduction slots. Returns a graph whose
        `launches` counts one interval; the caller adds the passes run."""
        ctx = ctypes.c_void_p()
        before = self.launches
        self.lib.call("gridlp_loop_graph_begin", self.stream(), ctypes.byref(ctx))
        try:
            build()
            self.lib.call("gridlp_loop_graph_decide", ctx, self.slots.data_ptr(), loop_dev.data_ptr(),
                          ring_dev.data_ptr())
        except BaseException:
            self.lib._lib.gridlp_loop_graph_abort(ctx)
            self.launches = before
            raise
        h = ctypes.c_void_p()
        per_interval = self.launches - before + 1
        self.launches = before
        self.lib.call("gridlp_loop_graph_end", ctx, ctypes.byref(h))
        return _IterateGraph(self, h, per_interval)

    def cluster_plan(self, psrc, dsrc):
        """gridlp_cluster_plan for a matrix pair: the host plan array, or None
        when the LP does not fit one cluster (GRIDLP_ERR_UNSUPPORTED)."""
        plan = (ctypes.c_int64 * native.CLUSTER_PLAN_LEN)()
        rc = self.lib._lib.gridlp_cluster_plan(self.src(psrc), self.src(dsrc), plan, native.CLUSTER_PLAN_LEN)
        if rc == 4:
            return None
        if rc != 0:
            raise native.GridlpError(f"gridlp_cluster_plan failed ({rc}): {self.lib.last_error()}")
        return plan

    def iterate_cluster(self, psrc, col, dsrc, row, count: int, halpern: bool, plan, kkt=None):
        """count fused iterations of a tiny single-block LP in one cluster
        launch (gridlp_pdhg_iterate_cluster) with a plan of cluster_plan();
        `kkt` (native.ClusterKkt) fuses the closing KKT / probe pass."""
        self.lib.call("gridlp_pdhg_iterate_cluster", self.src(psrc), self.primal_struct(col), self.src(dsrc),
                      self.dual_struct(row), self.step.data_ptr(), int(count), _pflags(col, halpern), plan,
                      ctypes.byref(kkt) if kkt is not None else None, self.stream())
        self.launches += 1 if (count or kkt is not None) else 0

    def reduce_terms(self, terms, n: int, nred: int, slot: int):
        """gridlp_reduce_terms: the canonical reduction of per-row terms into
        a reduction slot."""
        self.launches += 2
        self.lib.call("gridlp_reduce_terms", terms.data_ptr(), int(n), int(nred), self.red(slot), self.stream())

    def step_advance(self, delta: int):
        self.launches += 1
        self.lib.call("gridlp_op_step_advance", self.step.data_ptr(), int(delta), self.stream())
