"""PDHG engine: restarted Halpern PDHG over an R x C grid of HBM-resident
blocks, driving the sm_100a kernels of libgridlp_b200.so.

Reference: iterate_epoch and its helpers (/root/reference/pkg/src/gridlp/
pdhg_engine.py:223-476) and the step-size setup of solve()
(solver_driver.py:211-234, sparse_kernels.py:61-93).

Per main-loop iteration, per grid column j and row i:
  primal:  [Aᵀy]_j -> x̂, x̄, Halpern x   (one fused kernel when R == 1)
  dual:    [A x̄]_i -> ŷ, Halpern y        (one fused kernel when C == 1)
When the reduced axis is longer than one, each block writes its partial
product and the epilogue kernel consumes the axis sum (ascending-order sum of
the resident partials on one GPU, or an NCCL allreduce across GPUs).
A chunk of iterations up to the next KKT pass is captured once as a CUDA
graph and replayed; the Halpern counter lives on the device and the graph
advances it itself.

Every restart / termination decision is taken on the host from scalars
reduced in the reference's order (ascending device rank), exactly as
pdhg_engine.py:405-462 does, with the same collective ledger.
"""

from __future__ import annotations

import ctypes
import dataclasses
import logging
import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from .blocks import (DEFAULT_EXACT_ROW_MAX, DEFAULT_LIGHT_ROW_MAX, LIGHT_ROW_CANDIDATES, BandedCsr,
                     split_column_bands, BandSetup, DeviceCsr, DeviceSetup, inverse_order,
                     inverse_order_device, length_order, length_order_device, permute_csr, permute_matrix,
                     slice_blocks, transpose, upload)
from . import native
from .comm import Ledger, asc_sum
from .ops import Fused, Parts, PeerDest, PeerSrc

log = logging.getLogger("gridlp.solver")

OPTIMAL = "optimal"
ITERATION_LIMIT = "iteration_limit"
TIME_LIMIT = "time_limit"
NUMERICAL_FAILURE = "numerical_failure"

# per-coord scalar table fields of one KKT pass
F_RP2, F_PEN, F_RD2, F_CX, F_RCX, F_DX2, F_DY2, F_CROSS, F_TIME = range(9)
NFIELDS = 9


ORDER_WINDOW_ROWS = 4096      # locality window of _choose_order
ORDER_LOCALITY_RATIO = 2.0    # layout order when its window span is <= 1/2 of the class order's


@dataclass
class EngineOptions:
    """EngineConfig (pdhg_engine.py:138-154) plus device knobs."""

    tolerance: float = 1e-4
    max_iterations: int = 100_000
    kkt_interval: int = 64
    gamma: float = 0.0
    halpern: bool = True
    restarts: bool = True
    beta_sufficient: float = 0.2
    beta_necessary: float = 0.8
    beta_artificial: float = 0.36
    pid_kp: float = 0.6
    pid_ki: float = 0.1
    pid_kd: float = 0.1
    omega_min: float = 1e-6
    omega_max: float = 1e6
    time_limit_seconds: float | None = None
    exact_row_max: int = DEFAULT_EXACT_ROW_MAX   # rows up to this length: sequential (bit-exact) sums
    # rows up to this length: SELL-32 lanes; None = per block, the fastest of
    # LIGHT_ROW_CANDIDATES by a timed product (device setup). Result-neutral:
    # products are bit-identical and fused reductions are summed in a fixed
    # row order (gridlp_red_t.terms), so the choice may vary between runs
    light_row_max: int | None = None
    # internal length-class row/column order per band (CUDA only); None = the
    # class order unless the layout order has 2x better gather locality
    # (deterministic statistic, PdhgEngine._choose_order)
    sorted_order: bool | None = None
    # inside each column class, columns in first-touch order of the A
    # products (device setup, class order): coalesced first gathers
    first_touch_cols: bool = True
    # column bands per block (BandedCsr): None = when the gather vector of a
    # block exceeds band_bytes, ceil(bytes / band_bytes) bands if a timed
    # product says so; an int forces that many (1 = never). Bit-identical.
    column_bands: int | None = None
    band_bytes: int = 48 << 20
    # blocks above this many nonzeros skip the timed column-band choice (the
    # torch-level band split needs ~40 B/nnz of temporaries: a 2B-nnz block
    # of cfg5 on a 2x2 grid would not fit next to its own SELL copy)
    band_max_nnz: int = 1 << 30
    # band problems on the single-process grid: length-class order from a
    # counting pass over the generated blocks (False: layout order)
    band_class_order: bool = True
    # value storage per block (gridlp_csr_t.val_codec): "auto" = the
    # narrowest LOSSLESS codec of the block's values (+-1 only: sign bit in
    # the column index, 4 B/nnz; all exactly float: 8 B/nnz; else FP64,
    # 12 B/nnz) for blocks of at least value_codec_min_nnz nonzeros (smaller
    # blocks sit in L2 / in one cluster's shared memory, where the bytes do
    # not matter and the cluster launch needs FP64); "f64" = always FP64.
    # Products are bit-identical either way.
    value_codec: str = "auto"
    value_codec_min_nnz: int = 1 << 20
    device_setup: bool = True
    use_graphs: bool = True
    # capture the NCCL executor's iterations (kernels + NCCL collectives) in
    # a CUDA graph too, as the single-GPU and peer executors do
    graph_nccl: bool = True
    graph_chunk: int = 128
    # single-block LPs up to this many nonzeros run each chunk of iterations
    # as ONE cooperative launch with grid barriers between the products
    # (gridlp_pdhg_iterate_persistent, bit-identical iterates); 0 = never.
    # Off by default: measured slower than the chained CUDA-graph path at
    # every size (cfg1 8.96 vs 7.25 µs/iteration, profiles/r2/README.md) —
    # two global-memory grid barriers per iteration cost more than the
    # kernel boundaries PDL already hides
    persistent_max_nnz: int = 0
    # single-block solves: the main loop runs on the device — one CUDA graph
    # with a WHILE node whose body is a KKT interval (iterations, pass, and a
    # one-thread kernel evaluating the reference's termination / restart
    # logic on the pass's slots), so intervals follow each other without a
    # host round trip; the host replays each pass's bookkeeping afterwards
    # and handles restarts (gridlp_loop_graph_*). Bit-identical iterates
    # and decisions (checked pass by pass). Opt-in: a conditional body
    # loses the programmatic chaining of the kernel-per-product chunks
    # (cfg2: 12.0 vs 11.2 ms per interval, e2e equal), and on the cluster
    # launch (cfg1) it is faster on average but bimodal (0.087-0.098 s and
    # 0.088-0.116 s vs a steady 0.095 s host-driven); None = cluster-launched
    # LPs only, True = every single-block LP, False = never (default).
    device_loop: bool | None = False
    device_loop_passes: int = 1024
    # tiny single-block LPs (vectors + matrix within one 8-CTA cluster's
    # shared memory, e.g. BASELINE configs[0]) run each chunk of iterations
    # in one thread-block-cluster launch (gridlp_pdhg_iterate_cluster,
    # bit-identical iterates); falls back by itself when the LP is too big
    cluster_small: bool = True
    # with the cluster launch, the chunk's closing KKT / probe pass runs in the
    # same launch (only the canonical term reductions follow)
    cluster_fused_pass: bool = True
    # NCCL executor, main loop: each axis sum is an ordered reduce-scatter
    # (all-to-all of the partial shards, then the epilogue adds the G member
    # slices in ascending order — the reference's order, comm.py:75-84) and
    # the epilogue runs on this rank's 1/G shard only; the updated x_bar / y
    # shard is all-gathered. Same NVLink bytes as an allreduce, 1/G of the
    # epilogue bytes, bit-identical to the virtual grid. False: allreduce
    # (NCCL's order) + replicated epilogue.
    nccl_sharded: bool = True


@dataclass
class ColState:
    j: int
    n: int
    c: torch.Tensor
    lo: torch.Tensor
    hi: torch.Tensor
    x: torch.Tensor
    xbar: torch.Tensor
    x0: torch.Tensor
    xpb: torch.Tensor
    v: torch.Tensor
    s: torch.Tensor
    scale: torch.Tensor | None = None     # Dc of a scaled LP (KKT on the original LP)
    uniform_bounds: bool = False          # every variable bounded by lo[0], hi[0] (GRIDLP_F_UNIFORM_BOUNDS)


@dataclass
class RowState:
    i: int
    m: int
    lo: torch.Tensor
    hi: torch.Tensor
    y: torch.Tensor
    y0: torch.Tensor
    ax: torch.Tensor
    dy: torch.Tensor
    u: torch.Tensor
    scale: torch.Tensor | None = None     # Dr of a scaled LP


@dataclass
class ShardPlan:
    """One axis sum of the sharded NCCL executor (PdhgEngine._shard_plan)."""

    axis: str
    index: int
    src: object          # Fused product of the local block
    partial: torch.Tensor
    recv: torch.Tensor
    final: object        # Parts over the G received slices of this rank's shard
    state: object        # ColState / RowState view of the shard
    me: int
    S: int
    G: int


@dataclass
class BlockState:
    i: int
    j: int
    A: DeviceCsr
    AT: DeviceCsr
    bufs: dict = field(default_factory=dict)


@dataclass
class Report:
    r_primal: float
    r_dual: float
    r_gap: float
    obj_primal: float
    obj_dual: float

    @property
    def overall(self) -> float:
        return max(self.r_primal, self.r_dual, self.r_gap)


class nvtx_range:
    """NVTX range around a solve phase (setup, power iteration, iterations,
    KKT pass), visible to ncu --nvtx / nsys; nothing when CUDA is absent."""

    def __init__(self, name: str):
        self.name = name
        self.on = torch.cuda.is_available()

    def __enter__(self):
        if self.on:
            torch.cuda.nvtx.range_push(self.name)
        return self

    def __exit__(self, *exc):
        if self.on:
            torch.cuda.nvtx.range_pop()
        return False


def gap_residual(p: float, d: float) -> float:
    """pdhg_engine.py:211-216."""
    if not math.isfinite(d) or not math.isfinite(p):
        return float("inf")
    return abs(p - d) / (1.0 + max(abs(p), abs(d)))


def restart_decision(base, r_current, r_prev, inner_k, total, bs, bn, ba) -> bool:
    """pdhg_engine.py:262-282."""
    if base is not None:
        if r_current <= bs * base:
            return True
        if r_prev is not None and r_current <= bn * base and r_current > r_prev:
            return True
    return inner_k >= ba * total


class Pid:
    """pdhg_engine.py:97-103, :285-307."""

    def __init__(self, kp, ki, kd):
        self.kp, self.ki, self.kd = kp, ki, kd
        self.integral = 0.0
        self.last_error = 0.0

    def update(self, d_x, d_y, omega, lo, hi) -> float:
        if d_x <= 0.0 or d_y <= 0.0:
            return omega
        so = math.sqrt(omega)
        err = math.log((so * d_x) / (d_y / so))
        self.integral += err
        lw = math.log(omega) - (self.kp * err + self.ki * self.integral + self.kd * (err - self.last_error))
        self.last_error = err
        return min(max(math.exp(lw), lo), hi)


def _broken(rep: Report) -> bool:
    """pdhg_engine.py:356-361."""
    return (not math.isfinite(rep.r_primal)) or (not math.isfinite(rep.r_dual)) or math.isnan(rep.obj_primal)


class PdhgEngine:
    """Blocks, state and the main loop for the coords local to this process."""

    def __init__(self, problem, layout, opts: EngineOptions, comm, ops_factory, device,
                 objective_norm: float, bound_norm: float, objective_constant: float, preload=None,
                 kkt_scale=None):
        self.opts = opts
        self.layout = layout
        self.comm = comm
        self.device = device
        self.R, self.C = layout.topology.rows, layout.topology.cols
        self.cnorm, self.bnorm, self.const = objective_norm, bound_norm, objective_constant
        self.ledger = Ledger()
        self.timings = {}
        self._ops_factory = ops_factory
        self.choices = {}
        t0 = time.perf_counter()
        self._kkt_scale = kkt_scale      # (Dr, Dc) user-order device vectors of a scaled LP, or None
        self._build(problem, preload)
        if comm.kind == "peer":
            (i0, j0), = comm.local
            comm.setup_axes(self.rows[i0].m, self.cols[j0].n)
        self.timings["setup_blocks_s"] = time.perf_counter() - t0
        cap = max([b.A.slots() for b in self.blocks.values()]
                  + [b.AT.slots() for b in self.blocks.values()] + [1184])
        self.nslots = self._assign_slots()
        self.ops = ops_factory(device, cap, self.nslots)
        if hasattr(self.ops, "enable_terms"):
            # reductions independent of the layout choices (row classes, bands)
            self.ops.enable_terms(max([b.A.num_rows for b in self.blocks.values()]
                                      + [b.AT.num_rows for b in self.blocks.values()] + [1]))
        self._plans()
        self._graph = None
        self._graph_launches = 0
        self.iteration_events = None   # bench hook: list of (start, end, iterations)

    # ------------------------------------------------------------ setup
    def _build(self, problem, preload=None):
        lay, dev = self.layout, self.device
        banded = hasattr(problem, "bands")       # blocks generated per device (synth.BandProblem)
        on_device = dev.type == "cuda" and (self.opts.device_setup or banded)
        tm = self.timings
        if on_device:
            t0 = time.perf_counter()
            setup = BandSetup(problem, lay, dev) if banded else DeviceSetup(problem, lay, dev, preload)
            torch.cuda.synchronize(dev)
            tm["setup_upload_s"] = time.perf_counter() - t0
            tm.update(getattr(setup, "times", {}))
            self.setup_h2d_bytes = setup.h2d_bytes
            host_blocks = None
        else:
            pa = permute_matrix(problem.matrix, lay)
            host_blocks = slice_blocks(pa, lay)
            self.per_device_nnz = [host_blocks[c].nnz for c in lay.topology.coords()]
            self.setup_h2d_bytes = 0
        cp, rp = lay.perm.col_perm, lay.perm.row_perm
        t0 = time.perf_counter()
        # a band problem's row lengths are only known per block, and ranks sharing
        # a band must agree on its order, so across processes it keeps the layout
        # order; on the single-process grid every block is local: a counting pass
        # over the generated blocks gives the class order (_band_orders)
        if banded and on_device and self.comm.kind == "virtual" and self.opts.sorted_order is not False \
                and self.opts.band_class_order:
            self._band_orders(setup)
        else:
            self._internal_orders(problem, dev.type == "cuda" and self.opts.sorted_order is not False and not banded,
                                  setup if on_device else None)
        tm["setup_orders_s"] = time.perf_counter() - t0
        if on_device and not banded and self.sorted and self.opts.sorted_order is None:
            t0 = time.perf_counter()
            self._choose_order(setup)
            tm["setup_order_choice_s"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        f64 = dict(dtype=torch.float64, device=dev)
        # with the device setup the vectors go up in the user's order and one
        # device gather per band applies layout permutation + internal order
        # (the composed index is kept for the solution's way back)
        dev_vec = on_device and not banded
        self._col_idx, self._row_idx = {}, {}
        if dev_vec:
            cpd = setup.col_perm[:lay.num_cols].long()
            rpd = setup.row_perm[:lay.num_rows]
            obj, vlo, vhi, clo, chi = (upload(np.asarray(getattr(problem, k)), np.float64, dev) for k in
                                       ("objective", "var_lower", "var_upper", "con_lower", "con_upper"))
        elif not banded:
            obj = np.asarray(problem.objective, np.float64)[cp]
            vlo = np.asarray(problem.var_lower, np.float64)[cp]
            vhi = np.asarray(problem.var_upper, np.float64)[cp]
            clo = np.asarray(problem.con_lower, np.float64)[rp]
            chi = np.asarray(problem.con_upper, np.float64)[rp]
        local = self.comm.local
        self.local_cols = sorted({j for _, j in local})
        self.local_rows = sorted({i for i, _ in local})
        self.sharded = (self.comm.kind == "nccl" and self.opts.nccl_sharded and hasattr(self.comm, "exchange")
                        and (self.R > 1 or self.C > 1))

        def padded(length, group):
            """zeros(length) as a view of storage padded to group * ceil(length / group)
            (the all-gather of the shards writes into it in place)"""
            if not self.sharded or group <= 1:
                return torch.zeros(length, **f64)
            S = -(-length // group)
            return torch.zeros(max(group * S, 1), **f64)[:length]
        self.cols, self.rows, self.blocks = {}, {}, {}
        for j in self.local_cols:
            c0, c1 = lay.col_range(j)
            n = c1 - c0
            t = lambda a: self._to_internal_col(j, a[c0:c1])  # noqa: E731
            if dev_vec:
                idx = cpd[c0:c1]
                if self.sorted:
                    idx = idx[self.col_order[j].long()]
                self._col_idx[j] = idx
                t = lambda a: a[idx]  # noqa: E731
            if banded:
                cj, lj, hj, _ = problem.bands.col_data(c0, c1)
                t = (lambda a, o=self.col_order[j].long(): a[o]) if self.sorted else (lambda a: a)  # noqa: E731
                obj, vlo, vhi = cj, lj, hj
            self.cols[j] = ColState(j, n, t(obj), t(vlo), t(vhi), padded(n, self.R),
                                    padded(n, self.R), torch.zeros(n, **f64),
                                    torch.zeros(n, **f64), torch.zeros(n, **f64),
                                    torch.zeros(n, **f64),
                                    t(self._kkt_scale[1] if dev_vec else self._kkt_scale[1].cpu().numpy())
                                    if self._kkt_scale is not None else None)
        for i in self.local_rows:
            r0, r1 = lay.row_range(i)
            m = r1 - r0
            t = lambda a: self._to_internal_row(i, a[r0:r1])  # noqa: E731
            if dev_vec:
                idx = rpd[r0:r1]
                if self.sorted:
                    idx = idx[self.row_order[i].long()]
                self._row_idx[i] = idx
                t = lambda a: a[idx]  # noqa: E731
            if banded:
                li, hi_, _ = problem.bands.row_data(r0, r1)
                t = (lambda a, o=self.row_order[i].long(): a[o]) if self.sorted else (lambda a: a)  # noqa: E731
                clo, chi = li, hi_
            self.rows[i] = RowState(i, m, t(clo), t(chi), padded(m, self.C), torch.zeros(m, **f64),
                                    torch.zeros(m, **f64), torch.zeros(m, **f64), torch.zeros(m, **f64),
                                    t(self._kkt_scale[0] if dev_vec else self._kkt_scale[0].cpu().numpy())
                                    if self._kkt_scale is not None else None)
        for col in self.cols.values():
            if col.n and col.lo.is_cuda:
                col.uniform_bounds = bool(torch.equal(col.lo, col.lo[:1].expand(col.n))
                                          and torch.equal(col.hi, col.hi[:1].expand(col.n)))
        kw = dict(exact_row_max=self.opts.exact_row_max,
                  light_row_max=self.opts.light_row_max if self.opts.light_row_max is not None
                  else DEFAULT_LIGHT_ROW_MAX)
        tm["setup_vectors_s"] = time.perf_counter() - t0
        nnz_of = {}
        for (i, j) in local:
            if on_device:
                t0 = time.perf_counter()
                a = setup.block(i, j)
                torch.cuda.synchronize(dev)
                t1 = time.perf_counter()
                at = setup.transpose(a)
                torch.cuda.synchronize(dev)
                tm["setup_transpose_only_s"] = tm.get("setup_transpose_only_s", 0.0) + time.perf_counter() - t1
                if self.sorted:
                    # internal order: A_ij rows by sigma_i, columns by tau_j (and the
                    # transpose's the other way round); the transpose is taken first
                    # so its entries stay in layout row order (row sums unchanged)
                    d32 = lambda o: o.to(torch.int32) if isinstance(o, torch.Tensor) else torch.from_numpy(  # noqa: E731
                        o.astype(np.int32)).to(dev)
                    a = setup.permute(a, d32(self.row_order[i]), d32(self.col_inv[j]))
                    at = setup.permute(at, d32(self.col_order[j]), d32(self.row_inv[i]))
                torch.cuda.synchronize(dev)
                t2 = time.perf_counter()
                da = self._block_auto(setup, a, self.col_order[j] if self.sorted else None)
                del a                   # each CSR input goes as soon as its SELL copy exists (peak HBM)
                a = None
                dt = self._block_auto(setup, at, self.row_order[i] if self.sorted else None)
                at = None
                torch.cuda.synchronize(dev)
                t3 = time.perf_counter()
                tm["setup_extract_s"] = tm.get("setup_extract_s", 0.0) + t1 - t0
                tm["setup_transpose_s"] = tm.get("setup_transpose_s", 0.0) + t2 - t1
                tm["setup_sell_s"] = tm.get("setup_sell_s", 0.0) + t3 - t2
                del a, at
                self.blocks[(i, j)] = BlockState(i, j, da, dt)
                nnz_of[(i, j)] = self.blocks[(i, j)].A.nnz
            else:
                hb = host_blocks[(i, j)]
                ht = transpose(hb)
                if self.sorted:
                    ho = self._host_order
                    hb = permute_csr(hb, ho(self.row_order[i]), ho(self.col_inv[j]))
                    ht = permute_csr(ht, ho(self.col_order[j]), ho(self.row_inv[i]))
                self.blocks[(i, j)] = BlockState(i, j, DeviceCsr(hb, dev, value_codec=self._codec_for(hb.nnz), **kw),
                                                 DeviceCsr(ht, dev, value_codec=self._codec_for(ht.nnz), **kw))
        if on_device:
            t0 = time.perf_counter()
            setup.release()     # the freed setup buffers stay in torch's caching allocator for reuse
            del setup
            tm["setup_release_s"] = time.perf_counter() - t0
            coords = lay.topology.coords()
            if self.comm.kind == "virtual":
                self.per_device_nnz = [nnz_of.get(c, -1) for c in coords]
            else:      # one block per rank: gather the counts (same sequence on every rank)
                tab = self.comm.table({c: np.array([float(v)]) for c, v in nnz_of.items()})
                self.per_device_nnz = [int(tab[c][0]) for c in coords]
        del host_blocks
        self._trial_ops = None
        self.choices.setdefault("order", "sorted" if self.sorted else "layout")
        self.choices["light_row_max"] = {f"{k}{i},{j}": getattr(b, k).light_row_max
                                         for (i, j), b in self.blocks.items() for k in ("A", "AT")}
        self.choices["column_bands"] = {f"{k}{i},{j}": len(getattr(getattr(b, k), "bands", [None]))
                                        for (i, j), b in self.blocks.items() for k in ("A", "AT")}
        self.choices["value_codec"] = {
            f"{k}{i},{j}": ",".join(sorted({d.codec for d in getattr(getattr(b, k), "bands", [getattr(b, k)])}))
            for (i, j), b in self.blocks.items() for k in ("A", "AT")}
        self._banded = any(isinstance(m, BandedCsr) for b in self.blocks.values() for m in (b.A, b.AT))
        tensors = [t for b in self.blocks.values() for d in (b.A, b.AT) for t in d.tensors()]
        tensors += [t for c in self.cols.values() for t in (c.c, c.lo, c.hi)]
        tensors += [t for r in self.rows.values() for t in (r.lo, r.hi)]
        self.h2d_bytes = int(sum(t.numel() * t.element_size() for t in tensors))
        if self.setup_h2d_bytes:      # blocks were built on the device from the uploaded CSR
            self.h2d_bytes = int(self.setup_h2d_bytes + sum(
                t.numel() * t.element_size() for c in self.cols.values() for t in (c.c, c.lo, c.hi))
                + sum(t.numel() * t.element_size() for r in self.rows.values() for t in (r.lo, r.hi)))
        self.passes = 0

    # ------------------------------------------------- layout choices
    def _codec_for(self, nnz: int) -> str:
        o = self.opts
        return o.value_codec if nnz >= o.value_codec_min_nnz else "f64"

    def _sell_csr(self, setup, arr, light: int) -> DeviceCsr:
        d = setup.sell(arr, light)
        d["shape"] = (arr.num_rows, arr.num_cols, arr.nnz)
        return DeviceCsr(d, self.device, exact_row_max=self.opts.exact_row_max, light_row_max=light,
                         value_codec=self._codec_for(arr.nnz))

    def _time_products(self, mats) -> float:
        """Median device time of one product with each matrix (summed), on
        random gather vectors: the cost model of the layout choices."""
        dev = self.device
        need = max(m.slots() for m in mats) + 8
        ops = getattr(self, "_trial_ops", None)
        if ops is None or ops.capacity < need:
            ops = self._trial_ops = self._ops_factory(dev, max(need, 4096), 1)
        gen = torch.Generator(device=dev)
        gen.manual_seed(0)
        xs = [torch.rand(max(m.num_cols, 1), dtype=torch.float64, device=dev, generator=gen)[:m.num_cols]
              for m in mats]
        outs = [torch.empty(m.num_rows, dtype=torch.float64, device=dev) for m in mats]

        def run():
            for m, x, o in zip(mats, xs, outs):
                ops.store(Fused(m, x), o)
        run()
        times = []
        for _ in range(5):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            run()
            e1.record()
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        # the trial ops cache one C source per Fused object (matrix + gather
        # vector): drop them, so a losing candidate's HBM is freed as soon as
        # the caller lets go of it
        ops._srcs.clear()
        del xs, outs
        return sorted(times)[2] * 1e-3

    def _sell_auto(self, setup, arr) -> DeviceCsr:
        """SELL-32 layout of one block (or transpose). With light_row_max set
        it is used as is; otherwise rows of length (128, 2048] may go to the
        SELL lanes instead of the warp-per-row path when a timed product says
        so (lanes walk consecutive rows, so when neighbouring rows gather
        neighbouring columns — multi-commodity coupling rows — their gathers
        coalesce; on power-law rows the warp-per-row path is faster)."""
        if self.opts.light_row_max is not None:
            return self._sell_csr(setup, arr, self.opts.light_row_max)
        cands = [DEFAULT_LIGHT_ROW_MAX]
        if arr.num_rows and arr.nnz:
            lens = arr.ptr[1:] - arr.ptr[:-1]
            for lo, hi in zip(LIGHT_ROW_CANDIDATES, LIGHT_ROW_CANDIDATES[1:]):
                if bool(((lens > lo) & (lens <= hi)).any()):
                    cands.append(hi)
        if len(cands) == 1:
            return self._sell_csr(setup, arr, cands[0])
        best, best_t = None, None
        for light in cands:
            d = self._sell_csr(setup, arr, light)
            t = self._time_products([d])
            if best_t is None or t < 0.97 * best_t:
                best, best_t = d, t
            del d
        return best

    def _block_auto(self, setup, arr, to_layout=None):
        """_sell_auto, then column bands (BandedCsr) when the block's gather
        vector is larger than band_bytes and banding is measured faster (or
        forced by column_bands): each band's slice of x̄ / y then stays in
        L2 instead of every gather being a DRAM sector. Bands are layout
        column ranges (`to_layout` maps the length-class order back), along
        which every row's entries ascend, so a band is a contiguous piece of
        each row's add chain."""
        best = self._sell_auto(setup, arr)
        o = self.opts
        if o.column_bands is None and arr.nnz > o.band_max_nnz:
            return best
        cuts = self._band_cuts(arr.num_cols) if arr.nnz or o.column_bands is not None else [0, arr.num_cols]
        K = len(cuts) - 1
        if K <= 1:
            return best
        parts = split_column_bands(arr, cuts, o.exact_row_max, to_layout)
        banded = BandedCsr([self._sell_auto(setup, p) for p in parts], cuts, self.device)
        del parts
        if o.column_bands is not None:
            return banded
        # result-neutral choice: take bands when they measure >= 1 % faster
        if self._time_products([banded]) < 0.99 * self._time_products([best]):
            return banded
        return best

    def _choose_order(self, setup):
        """sorted_order=None: keep the length-class order unless the layout
        order has much better gather locality — the median column span of
        ORDER_WINDOW_ROWS consecutive rows (128 SELL slices, about what the
        GPU works on at once) in the layout order is at most half the span in
        the class order (random and power-law matrices: ratio ~1.0; MCF 2.7-7). Block-structured matrices (multi-commodity
        flow: one commodity's rows and columns together) keep the layout
        order; each length class would sweep all commodities, re-reading x̄
        from DRAM once per class. A pure function of the matrix and layout,
        so every run and every rank decides alike (the two orders differ in
        reduction rounding, not in products)."""
        lay = self.layout
        m, nnz = lay.num_rows, setup.nnz
        if m == 0 or nnz == 0:
            self.choices["order"] = "sorted"
            return
        dev = self.device
        ptr = setup.src_ptr
        lens = ptr[1:] - ptr[:-1]
        rid = torch.repeat_interleave(torch.arange(m, device=dev), lens)
        lc = setup.inv_col[setup.src_col[:nnz].long()].long()
        big = lay.num_cols + 1
        rmin = torch.full((m,), big, dtype=torch.int64, device=dev).scatter_reduce(0, rid, lc, "amin")
        rmax = torch.full((m,), -1, dtype=torch.int64, device=dev).scatter_reduce(0, rid, lc, "amax")
        del rid, lc

        def median_span(seq, w=ORDER_WINDOW_ROWS):
            pad = (-seq.numel()) % w
            mn = torch.cat([rmin[seq], torch.full((pad,), big, dtype=torch.int64, device=dev)]).view(-1, w)
            mx = torch.cat([rmax[seq], torch.full((pad,), -1, dtype=torch.int64, device=dev)]).view(-1, w)
            smin, smax = mn.min(1).values, mx.max(1).values
            ok = smax >= 0
            return float((smax - smin)[ok].double().median().item()) if bool(ok.any()) else 0.0

        layout_seq = setup.row_perm[:m]
        sorted_seq = torch.cat([layout_seq[lay.row_range(i)[0]:lay.row_range(i)[1]][self.row_order[i].long()]
                                for i in range(self.R)])
        span_layout, span_sorted = median_span(layout_seq), median_span(sorted_seq)
        self.choices["order_spans"] = {"layout": span_layout, "sorted": span_sorted}
        if ORDER_LOCALITY_RATIO * span_layout <= span_sorted:
            self.choices["order"] = "layout"
            self.sorted = False
            self.row_order, self.row_inv, self.col_order, self.col_inv = {}, {}, {}, {}
        else:
            self.choices["order"] = "sorted"

    # ------------------------------------------------- internal order
    def _internal_orders(self, problem, enabled: bool, setup=None):
        """Per grid row band i, sigma_i = the band's rows by full row length
        (length classes, longest first, stable); per grid column band j,
        tau_j = the band's columns by column count. Blocks and vectors live
        in this order on the device, so every SELL-32 slice holds rows of
        nearly equal length; entry order inside a row is untouched, so
        products stay bit-identical and iterates are the reference's up to
        the permutation. With the device setup the orders are computed and
        kept on the device (row lengths from the uploaded row pointers, column
        counts by histogram); every rank computes the same orders from the
        same problem."""
        self.sorted = bool(enabled)
        self.row_order, self.row_inv, self.col_order, self.col_inv = {}, {}, {}, {}
        if not self.sorted:
            return
        lay = self.layout
        if setup is not None:
            dev = self.device
            m, n = lay.num_rows, lay.num_cols
            row_len = (setup.src_ptr[1:] - setup.src_ptr[:-1])[setup.row_perm[:m]]
            col_len = setup.col_counts_device()[setup.col_perm[:n].long()] if n else row_len[:0]
            order, inverse = length_order_device, inverse_order_device
        else:
            A = problem.matrix
            row_len = np.diff(np.asarray(A.row_offsets, np.int64))[lay.perm.row_perm]
            col_len = np.bincount(A.col_indices, minlength=int(A.num_cols))[lay.perm.col_perm]
            order, inverse = length_order, inverse_order
        for i in range(self.R):
            r0, r1 = lay.row_range(i)
            self.row_order[i] = order(row_len[r0:r1])
            self.row_inv[i] = inverse(self.row_order[i])
        touch = self._first_touch(setup) if setup is not None and self.opts.first_touch_cols else None
        for j in range(self.C):
            c0, c1 = lay.col_range(j)
            if touch is None:
                self.col_order[j] = order(col_len[c0:c1])
            else:
                # first-touch order inside each length class (stable sorts:
                # by first touch, then by class)
                base = torch.sort(touch[c0:c1], stable=True).indices
                self.col_order[j] = base[length_order_device(col_len[c0:c1][base])]
            self.col_inv[j] = inverse(self.col_order[j])

    def _band_orders(self, setup):
        """Length-class order for a band problem on the single-process grid:
        one counting pass generates every block (deterministic, hash-based)
        for its row lengths and column counts, summed over the grid, then the
        blocks are generated again for the build. Cuts the layout order's
        SELL padding (planted rows: max of 32 near-binomial lengths)."""
        lay, dev = self.layout, self.device
        row_len = {i: torch.zeros(lay.row_range(i)[1] - lay.row_range(i)[0], dtype=torch.int64, device=dev)
                   for i in range(self.R)}
        col_len = {j: torch.zeros(lay.col_range(j)[1] - lay.col_range(j)[0], dtype=torch.int64, device=dev)
                   for j in range(self.C)}
        for i in range(self.R):
            for j in range(self.C):
                a = setup.block(i, j)
                row_len[i] += (a.ptr[1:] - a.ptr[:-1]).to(torch.int64)
                if a.nnz:
                    col_len[j] += torch.bincount(a.col[:a.nnz].long(), minlength=col_len[j].numel())
                del a
        self.sorted = True
        self.row_order, self.row_inv, self.col_order, self.col_inv = {}, {}, {}, {}
        for i in range(self.R):
            self.row_order[i] = length_order_device(row_len[i])
            self.row_inv[i] = inverse_order_device(self.row_order[i])
        for j in range(self.C):
            self.col_order[j] = length_order_device(col_len[j])
            self.col_inv[j] = inverse_order_device(self.col_order[j])
        self.choices["order"] = "sorted (band counting pass)"

    def _band_cuts(self, length: int) -> list:
        """Column-band cuts of a gather vector of `length` doubles: one band
        unless it exceeds band_bytes (or column_bands forces a count). (A
        band-major internal order — bands contiguous in HBM — was measured on
        cfg3 and did not pay: profiles/r2/README.md.)"""
        o = self.opts
        if o.column_bands is not None:
            K = int(o.column_bands)
        elif length * 8 > o.band_bytes:
            K = min(16, -(-length * 8 // o.band_bytes))
        else:
            K = 1
        K = max(1, min(K, max(length, 1)))
        return [(k * length) // K for k in range(K + 1)]

    def _first_touch(self, setup) -> torch.Tensor:
        """Per layout column, the position of its first use in the A
        products' SELL traversal (grid row band, slice, step, lane) under the
        internal row order. Ordering each column class by it gives the
        columns first gathered by one warp step consecutive ids, so those
        gathers coalesce (and, in Aᵀ, consecutive columns start at nearby
        rows). A column relabeling: products are unchanged bit for bit."""
        lay, dev = self.layout, self.device
        m, n, nnz = lay.num_rows, lay.num_cols, setup.nnz
        big = torch.iinfo(torch.int64).max
        if n == 0:
            return torch.zeros(0, dtype=torch.int64, device=dev)
        if m == 0 or nnz == 0:
            return torch.full((n,), big, dtype=torch.int64, device=dev)
        ptr = setup.src_ptr
        lens = ptr[1:] - ptr[:-1]
        internal_of_layout = torch.cat([lay.row_range(i)[0] + self.row_inv[i] for i in range(self.R)])
        inv_rp = torch.empty(m, dtype=torch.int64, device=dev)
        inv_rp[setup.row_perm[:m]] = torch.arange(m, dtype=torch.int64, device=dev)
        rank = internal_of_layout[inv_rp]                      # original row -> internal rank
        rid = torch.repeat_interleave(torch.arange(m, device=dev), lens)
        step = torch.arange(nnz, device=dev) - ptr[rid]
        rk = rank[rid]
        kmax = int(lens.max().item()) + 1
        key = ((rk // 32) * kmax + step) * 32 + (rk % 32)
        del rid, step, rk
        first = torch.full((n,), big, dtype=torch.int64, device=dev).scatter_reduce(
            0, setup.src_col[:nnz].long(), key, "amin")
        return first[setup.col_perm[:n].long()]                # layout order

    def _vec(self, a) -> torch.Tensor:
        """Host band slice -> FP64 device tensor (pinned staging on CUDA)."""
        if self.device.type == "cuda":
            return upload(a, np.float64, self.device)
        return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=self.device)

    @staticmethod
    def _take(v: torch.Tensor, order) -> torch.Tensor:
        idx = order if isinstance(order, torch.Tensor) else torch.as_tensor(order, device=v.device)
        return v[idx]

    @staticmethod
    def _place(v: torch.Tensor, order) -> np.ndarray:
        idx = order if isinstance(order, torch.Tensor) else torch.as_tensor(order, device=v.device)
        out = torch.empty_like(v)
        out[idx] = v
        return out.cpu().numpy()

    def _to_internal_col(self, j, a) -> torch.Tensor:
        v = self._vec(a)
        return self._take(v, self.col_order[j]) if self.sorted else v

    def _to_internal_row(self, i, a) -> torch.Tensor:
        v = self._vec(a)
        return self._take(v, self.row_order[i]) if self.sorted else v

    def _from_internal_col(self, j, v: torch.Tensor) -> np.ndarray:
        return self._place(v, self.col_order[j]) if self.sorted else v.cpu().numpy()

    def _from_internal_row(self, i, v: torch.Tensor) -> np.ndarray:
        return self._place(v, self.row_order[i]) if self.sorted else v.cpu().numpy()

    @staticmethod
    def _host_order(o) -> np.ndarray:
        return o.cpu().numpy() if isinstance(o, torch.Tensor) else o

    def _assign_slots(self):
        s = {}
        k = 0
        for i in self.local_rows:
            for name in ("kkt_rows", "probe", "anchor_y", "u"):
                s[(name, i)] = k
                k += 1
        for j in self.local_cols:
            for name in ("kkt_cols", "anchor_x", "v", "s"):
                s[(name, j)] = k
                k += 1
        for c in self.comm.local:
            s[("cross", c)] = k
            k += 1
        self.slot = s
        return k

    def _buf(self, blk, name, length):
        b = blk.bufs.get(name)
        if b is None:
            b = torch.zeros(length, dtype=torch.float64, device=self.device)
            blk.bufs[name] = b
        return b

    def _axis_plan(self, axis, index, items, length, keep, scratch_name):
        """items: [(block, orientation, gather)] of the local blocks on one grid
        row (C) / column (R), ascending. Returns (pre, reduce_args, final)."""
        single = (axis == "R" and self.R == 1) or (axis == "C" and self.C == 1)
        if single:
            (blk, orient, g), = items
            return [], None, Fused(blk.A if orient == "A" else blk.AT, g)
        if self.comm.kind == "peer":
            # fused exchange: the product writes into the group's receive slots,
            # the consumer adds them in slot order (no host collective)
            (blk, orient, g), = items
            local = self._buf(blk, f"{scratch_name}_{orient}", length) if keep else None
            return ([(Fused(blk.A if orient == "A" else blk.AT, g), PeerDest(self.comm.axes[axis], local))], None,
                    PeerSrc(self.comm.axes[axis], length))
        pre = []
        bufs = []
        for blk, orient, g in items:
            buf = self._buf(blk, f"{scratch_name}_{orient}", length)
            pre.append((Fused(blk.A if orient == "A" else blk.AT, g), buf))
            bufs.append(buf)
        if self.comm.kind == "virtual":
            return pre, None, Parts(bufs, length)
        scratch = None
        if keep:
            scratch = self._buf(items[0][0], f"{scratch_name}_red", length)
        target = scratch if keep else bufs[0]
        return pre, (axis, index, bufs, scratch), Parts([target], length)

    def _shard_plan(self, axis, index, items, vec_state, length):
        """Main-loop plan of the sharded NCCL executor on an axis of G > 1
        members (see EngineOptions.nccl_sharded): the block's partial product
        goes into a buffer padded to G * S, the all-to-all hands member q's
        slice of this rank's shard to recv[q], and the epilogue runs over the
        shard view of the vectors, adding the G slices in ascending order."""
        (blk, orient, g), = items
        G = self.R if axis == "R" else self.C
        me = self.comm.coord[0] if axis == "R" else self.comm.coord[1]
        S = -(-length // G)
        partial = self._buf(blk, f"sh_{axis}", G * S)
        recv = self._buf(blk, f"shr_{axis}", G * S)
        a = min(me * S, length)
        b = min(a + S, length)
        fields = [f.name for f in dataclasses.fields(vec_state)]
        view = {}
        for k in fields:
            v = getattr(vec_state, k)
            view[k] = v[a:b] if isinstance(v, torch.Tensor) else v
        view["n" if axis == "R" else "m"] = b - a
        shard_state = type(vec_state)(**view)
        return ShardPlan(axis, index, Fused(blk.A if orient == "A" else blk.AT, g), partial, recv,
                         Parts([recv[q * S:q * S + (b - a)] for q in range(G)], b - a), shard_state, me, S, G)

    def _plans(self):
        cols, rows, blocks = self.cols, self.rows, self.blocks
        col_items = lambda j, vec: [(blocks[(i, j)], "T", vec(i)) for i in self.local_rows if (i, j) in blocks]  # noqa: E731
        row_items = lambda i, vec: [(blocks[(i, j)], "A", vec(j)) for j in self.local_cols if (i, j) in blocks]  # noqa: E731
        self.plan_primal = {j: self._axis_plan("R", j, col_items(j, lambda i: rows[i].y), cols[j].n, False, "pT")
                            for j in self.local_cols}
        self.plan_dual = {i: self._axis_plan("C", i, row_items(i, lambda j: cols[j].xbar), rows[i].m, False, "pA")
                          for i in self.local_rows}
        self.plan_kkt_ax = {i: self._axis_plan("C", i, row_items(i, lambda j: cols[j].x), rows[i].m, True, "pAx")
                            for i in self.local_rows}
        self.plan_kkt_aty = {j: self._axis_plan("R", j, col_items(j, lambda i: rows[i].y), cols[j].n, False, "pT")
                             for j in self.local_cols}
        self.plan_probe = {i: self._axis_plan("C", i, row_items(i, lambda j: cols[j].xpb), rows[i].m, True, "pPr")
                           for i in self.local_rows}
        self.plan_pow_u = {i: self._axis_plan("C", i, row_items(i, lambda j: cols[j].v), rows[i].m, False, "pA")
                           for i in self.local_rows}
        self.plan_pow_s = {j: self._axis_plan("R", j, col_items(j, lambda i: rows[i].u), cols[j].n, False, "pT")
                           for j in self.local_cols}
        self.shard_primal, self.shard_dual = {}, {}
        if self.sharded:
            if self.R > 1:
                self.shard_primal = {j: self._shard_plan("R", j, col_items(j, lambda i: rows[i].y), cols[j],
                                                         cols[j].n) for j in self.local_cols}
            if self.C > 1:
                self.shard_dual = {i: self._shard_plan("C", i, row_items(i, lambda j: cols[j].xbar), rows[i],
                                                       rows[i].m) for i in self.local_rows}
        self._stale_x = False

    def _run_plan(self, plan):
        pre, red, final = plan
        for src, buf in pre:
            self.ops.store(src, buf)
        if red is not None:
            axis, index, bufs, scratch = red
            self.comm.reduce(axis, index, bufs, scratch)
        return final

    # ------------------------------------------------------- scalar tables
    def _table(self, local_vals: dict) -> dict:
        return self.comm.table(local_vals)

    def _axis_sum(self, table, field_, axis):
        """R: over i down my grid column; C: over j along my grid row."""
        i0, j0 = self.comm.local[0] if self.comm.local else (0, 0)
        if axis == "R":
            return asc_sum([table[(i, j0)][field_] for i in range(self.R)])
        return asc_sum([table[(i0, j)][field_] for j in range(self.C)])

    def _g_sum(self, table, field_, scale=1.0):
        return asc_sum([table[(i, j)][field_] / scale for i in range(self.R) for j in range(self.C)])

    # ---------------------------------------------------- power iteration
    def band_scalars(self):
        """(||c||, ||finite constraint bounds||) of a band problem from its
        device vectors: per band dot products (gridlp_op_dot), gathered once
        and summed in ascending band order (a band's vectors are replicated
        on its row / column of the grid, so each band is counted once)."""
        def sq(v, j_slot):
            fin = torch.where(torch.isfinite(v), v, torch.zeros_like(v))
            self.ops.dot(fin, fin, j_slot)
        for j, col in self.cols.items():
            sq(col.c, self.slot[("v", j)])
        vals = self.ops.read_slots(self.nslots)
        csq = {j: float(vals[self.slot[("v", j)], 0]) for j in self.cols}
        bsq = {}
        for i, row in self.rows.items():
            sq(row.lo, self.slot[("u", i)])
            lo_sq = float(self.ops.read_slots(self.nslots)[self.slot[("u", i)], 0])
            sq(row.hi, self.slot[("u", i)])
            bsq[i] = lo_sq + float(self.ops.read_slots(self.nslots)[self.slot[("u", i)], 0])
        tab = self._table({(i, j): np.array([csq[j], bsq[i]]) for (i, j) in self.comm.local})
        c_sq = asc_sum([tab[(0, j)][0] for j in range(self.C)])
        b_sq = asc_sum([tab[(i, 0)][1] for i in range(self.R)])
        return math.sqrt(c_sq), math.sqrt(b_sq)

    def power_estimate(self, iters: int, probe: np.ndarray | None, probe_seed: int = 0) -> float:
        """estimate_spectral_norm (sparse_kernels.py:61-93) on the grid.
        probe=None (band problems): each column band draws its own slice of a
        hash-based probe, u(seed, 31, j) in [-1, 1), on the device."""
        if iters < 1:
            raise ValueError("iters must be >= 1")
        ops, lay = self.ops, self.layout
        R, C = float(self.R), float(self.C)
        for j, col in self.cols.items():
            c0, c1 = lay.col_range(j)
            if probe is None:
                native.load().call("gridlp_gen_uniform", probe_seed, 31, c0, c1 - c0, -1.0, 1.0, col.v.data_ptr(),
                                   torch.cuda.current_stream(self.device).cuda_stream)
                if self.sorted:      # drawn in layout order: into the internal order
                    col.v.copy_(col.v[self.col_order[j].long()])
                continue
            col.v.copy_(self._to_internal_col(j, np.asarray(probe[c0:c1], dtype=np.float64)))
        if self.comm.kind == "virtual" and self.R == 1 and self.C == 1 and self.device.type == "cuda":
            return self._power_single_block(iters)
        est = 0.0
        for _ in range(iters):
            for i, row in self.rows.items():
                src = self._run_plan(self.plan_pow_u[i])
                ops.store(src, row.u, self.slot[("u", i)])
            for j, col in self.cols.items():
                ops.dot(col.v, col.v, self.slot[("v", j)])
            vals = ops.read_slots(self.nslots)
            local = {}
            for (i, j) in self.comm.local:
                row = np.zeros(2)
                row[0] = vals[self.slot[("u", i)], 0]
                row[1] = vals[self.slot[("v", j)], 0]
                local[(i, j)] = row
            tab = self._table(local)
            self.ledger.vec("C", "m")
            self.ledger.scalar("G", 2)
            u_sq = self._g_sum(tab, 0, C)
            v_sq = self._g_sum(tab, 1, R)
            if u_sq == 0.0 or v_sq == 0.0:
                return 0.0
            est = math.sqrt(u_sq / v_sq)
            for j, col in self.cols.items():
                src = self._run_plan(self.plan_pow_s[j])
                ops.store(src, col.s, self.slot[("s", j)])
            vals = ops.read_slots(self.nslots)
            local = {(i, j): np.array([vals[self.slot[("s", j)], 0]]) for (i, j) in self.comm.local}
            tab = self._table(local)
            self.ledger.vec("R", "n")
            self.ledger.scalar("G")
            s_sq = self._g_sum(tab, 0, R)
            if s_sq == 0.0:
                return est
            d = math.sqrt(s_sq)
            for col in self.cols.values():
                ops.div(col.s, col.v, d)
        return est

    def _power_single_block(self, iters: int) -> float:
        """power_estimate on a 1x1 grid without a host round trip per step:
        v = s / sqrt(s_sq) takes s_sq from its reduction slot on the device
        (gridlp_op_div_norm), each step's (u_sq, v_sq, s_sq) is copied to a
        device history, and the reference's early exits are replayed on the
        host from one read at the end. Steps after an early exit compute
        garbage that is never read; the estimate, the ledger and v are those
        of the step-by-step loop (v is only an internal probe)."""
        ops = self.ops
        row, col = self.rows[0], self.cols[0]
        su, sv, ss = self.slot[("u", 0)], self.slot[("v", 0)], self.slot[("s", 0)]
        pick = torch.tensor([su, sv, ss], dtype=torch.int64, device=self.device)
        hist = torch.empty((iters, 3), dtype=torch.float64, device=self.device)
        for k in range(iters):
            ops.store(self._run_plan(self.plan_pow_u[0]), row.u, su)
            ops.dot(col.v, col.v, sv)
            ops.store(self._run_plan(self.plan_pow_s[0]), col.s, ss)
            torch.index_select(ops.slots[:, 0], 0, pick, out=hist[k])
            ops.div_norm(col.s, col.v, ss)
        h = hist.cpu().numpy()
        est = 0.0
        for u_sq, v_sq, s_sq in h:
            self.ledger.vec("C", "m")
            self.ledger.scalar("G", 2)
            u_sq, v_sq, s_sq = float(u_sq) / 1.0, float(v_sq) / 1.0, float(s_sq) / 1.0
            if u_sq == 0.0 or v_sq == 0.0:
                return 0.0
            est = math.sqrt(u_sq / v_sq)
            self.ledger.vec("R", "n")
            self.ledger.scalar("G")
            if s_sq == 0.0:
                return est
        return est

    # -------------------------------------------------------- main loop
    def _persistent(self) -> bool:
        """Single block, no column bands, small enough to be launch bound."""
        if getattr(self, "_persist_ok", None) is None:
            nnz = sum(b.A.nnz for b in self.blocks.values())
            self._persist_ok = (self.R == 1 and self.C == 1 and hasattr(self.ops, "iterate_persistent")
                                and not self._banded and 0 < nnz <= self.opts.persistent_max_nnz)
        return self._persist_ok

    def _cluster_pass(self, mode: int, row, col):
        """gridlp_cluster_kkt_t for a chunk that ends at a KKT pass: the pass's
        per-row term buffers (allocated once) and the ax / x_probe_bar outputs."""
        t = getattr(self, "_pass_terms", None)
        if t is None:
            f64 = dict(dtype=torch.float64, device=self.device)
            t = self._pass_terms = {"rows": torch.zeros(4 * max(row.m, 1), **f64),
                                    "cols": torch.zeros(4 * max(col.n, 1), **f64),
                                    "probe": torch.zeros(2 * max(row.m, 1), **f64)}
        return native.ClusterKkt(mode, 0, t["rows"].data_ptr(), t["cols"].data_ptr(), t["probe"].data_ptr(),
                                 row.ax.data_ptr() if row.m else None, col.xpb.data_ptr() if col.n else None)

    def _cluster(self) -> bool:
        """Tiny single-block LP that fits one thread-block cluster: each
        chunk is one cluster launch (no graph; the plan is computed once,
        outside any capture)."""
        if getattr(self, "_cluster_ok", None) is None:
            ok = (self.opts.cluster_small and self.R == 1 and self.C == 1
                  and hasattr(self.ops, "cluster_plan") and not self._banded)
            self._cluster_plan = None
            if ok:
                (j, _), = self.cols.items()
                (i, _), = self.rows.items()
                self._cluster_plan = self.ops.cluster_plan(self.plan_primal[j][2], self.plan_dual[i][2])
            self._cluster_ok = self._cluster_plan is not None
        return self._cluster_ok

    def _launch_iterations(self, count: int):
        ops, h = self.ops, self.opts.halpern
        if self.R == 1 and self.C == 1 and hasattr(ops, "iterate") and count > 0 and not self._banded:
            # one block, fused sources: the whole chunk in one C-ABI call
            (j, col), = self.cols.items()
            (i, row), = self.rows.items()
            if self._cluster():
                mode = self.__dict__.pop("_fuse_pass_mode", 0)
                kkt = self._cluster_pass(mode, row, col) if mode else None
                try:
                    ops.iterate_cluster(self.plan_primal[j][2], col, self.plan_dual[i][2], row, count, h,
                                        self._cluster_plan, kkt)
                    if mode:
                        self._pass_in_launch = mode
                    return
                except native.GridlpError as exc:        # launch refused (e.g. no cluster scheduling)
                    log.warning("cluster launch refused (%s); using the kernel-per-product path", exc)
                    self._cluster_ok = False
            if self._persistent():
                if ops.iterate_persistent(self.plan_primal[j][2], col, self.plan_dual[i][2], row, count, h):
                    return
                self._persist_ok = False          # heavy rows: the graph path
            ops.iterate(self.plan_primal[j][2], col, self.plan_dual[i][2], row, count, h)
            return
        comm = self.comm
        for t in range(count):
            for j, col in self.cols.items():
                sp_ = self.shard_primal.get(j)
                if sp_ is None:
                    ops.primal(self._run_plan(self.plan_primal[j]), col, t, h)
                    continue
                ops.store(sp_.src, sp_.partial)
                comm.exchange(sp_.axis, j, sp_.partial, sp_.recv)
                ops.primal(sp_.final, sp_.state, t, h)
                comm.gather_shard(sp_.axis, j, col.xbar, sp_.me, sp_.S)
                self._stale_x = True        # x is current on this rank's shard only
            for i, row in self.rows.items():
                sd = self.shard_dual.get(i)
                if sd is None:
                    ops.dual(self._run_plan(self.plan_dual[i]), row, t, h)
                    continue
                ops.store(sd.src, sd.partial)
                comm.exchange(sd.axis, i, sd.partial, sd.recv)
                ops.dual(sd.final, sd.state, t, h)
                comm.gather_shard(sd.axis, i, row.y, sd.me, sd.S)
        ops.step_advance(count)

    def _sync_shards(self):
        """Sharded NCCL executor: all-gather x (updated on this rank's shard
        only during the main loop) before anything reads all of it — the KKT
        pass, a trace snapshot, the solution."""
        if not self._stale_x:
            return
        for j, col in self.cols.items():
            sp_ = self.shard_primal.get(j)
            if sp_ is not None:
                self.comm.gather_shard(sp_.axis, j, col.x, sp_.me, sp_.S)
        self._stale_x = False

    def _graphable(self) -> bool:
        if not (self.opts.use_graphs and self.device.type == "cuda"):
            return False
        return self.comm.kind in ("virtual", "peer") or (self.comm.kind == "nccl" and self.opts.graph_nccl
                                                          and getattr(self.comm, "graph_safe", False))

    def _run_iterations(self, count: int):
        if count <= 0:
            return
        ev = self.iteration_events
        if ev is not None:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            self._run_iterations_inner(count)
            e1.record()
            ev.append((e0, e1, count))
            return
        self._run_iterations_inner(count)

    def _run_iterations_inner(self, count: int):
        g = max(1, min(self.opts.graph_chunk, self.opts.kkt_interval))
        if not self._graphable() or count < g or self._persistent() or self._cluster():
            self._launch_iterations(count)
            return
        if self._graph is None:
            # warm every kernel once outside capture (the launch loads the
            # module), then capture while the GPU runs those iterations: no
            # synchronize before capture (torch.cuda.graph's context manager
            # would add one), so instantiation overlaps device work
            self._launch_iterations(g)
            count -= g
            if (self.R == 1 and self.C == 1 and not self._banded and hasattr(self.ops, "iterate_graph")):
                # one block: the whole chunk is one C-ABI call, captured in C
                # (no torch capture machinery, no synchronise, ~ms cheaper
                # per solve); the device keeps running the warm chunk meanwhile
                (j, col), = self.cols.items()
                (i, row), = self.rows.items()
                self._graph = self.ops.iterate_graph(self.plan_primal[j][2], col, self.plan_dual[i][2], row, g,
                                                     self.opts.halpern)
                self._graph_launches = 0            # the C graph counts its own launches
                while count >= g:
                    self._graph.replay()
                    count -= g
                if count:
                    self._launch_iterations(count)
                return
            stream = torch.cuda.Stream(self.device)
            graph = torch.cuda.CUDAGraph()
            before = getattr(self.ops, "launches", 0)
            if self.comm.kind == "nccl":
                # collectives inside a capture: fall back to eager launches if
                # this NCCL / driver combination refuses (never observed on one
                # rank; a multi-GPU first)
                torch.cuda.synchronize(self.device)
                try:
                    with torch.cuda.stream(stream):
                        graph.capture_begin()
                        try:
                            self._launch_iterations(g)
                        finally:
                            graph.capture_end()
                except RuntimeError as exc:
                    log.warning("CUDA-graph capture of the NCCL iterations failed (%s); running eager", exc)
                    self.opts.graph_nccl = False
                    torch.cuda.synchronize(self.device)
                    if count:
                        self._launch_iterations(count)   # captures do not execute: all remaining eagerly
                    return
            else:
                with torch.cuda.stream(stream):
                    graph.capture_begin()
                    try:
                        self._launch_iterations(g)
                    finally:
                        graph.capture_end()
            self._graph_launches = getattr(self.ops, "launches", 0) - before
            if hasattr(self.ops, "launches"):
                self.ops.launches = before     # capture records, it does not launch
            self._graph = graph
        while count >= g:
            self._graph.replay()
            if hasattr(self.ops, "launches") and self._graph_launches:
                self.ops.launches += self._graph_launches
            count -= g
        if count:
            self._launch_iterations(count)

    def _kkt(self, tau: float, restarts: bool):
        """One evaluation pass (+ the speculative restart probe). Returns
        (report, pieces) with host scalars reduced in the reference order."""
        self._kkt_launch(restarts)
        return self._kkt_collect(self.ops.read_slots(self.nslots), restarts)

    def _kkt_launch(self, restarts: bool):
        """The pass's device work (products, fused KKT / probe terms, slot
        reductions), no host read."""
        ops = self.ops
        self._sync_shards()
        fused_pass = self.__dict__.pop("_pass_in_launch", 0)
        if fused_pass and fused_pass == (2 if restarts else 1):
            # the cluster launch already computed the pass's per-row terms
            # (and ax, x_probe_bar): only the canonical reductions remain
            (i, row), = self.rows.items()
            (j, col), = self.cols.items()
            ops.reduce_terms(self._pass_terms["rows"], row.m, 4, self.slot[("kkt_rows", i)])
            ops.reduce_terms(self._pass_terms["cols"], col.n, 4, self.slot[("kkt_cols", j)])
            if restarts:
                ops.reduce_terms(self._pass_terms["probe"], row.m, 2, self.slot[("probe", i)])
            restarts_done = True
        else:
            restarts_done = False
        for i, row in ([] if restarts_done else self.rows.items()):
            src = self._run_plan(self.plan_kkt_ax[i])
            fused = isinstance(src, Fused)
            ops.kkt_rows(src, row, row.ax if fused else None, self.slot[("kkt_rows", i)])
        for j, col in ([] if restarts_done else self.cols.items()):
            src = self._run_plan(self.plan_kkt_aty[j])
            ops.kkt_cols(src, col, self.slot[("kkt_cols", j)])
        if restarts and not restarts_done:
            for i, row in self.rows.items():
                src = self._run_plan(self.plan_probe[i])
                if isinstance(src, Fused):
                    ops.probe(src, row, row.ax, None, self.slot[("probe", i)])
                else:
                    ops.probe(src, row, None, row.dy, self.slot[("probe", i)])
                    for j in self.local_cols:
                        blk = self.blocks.get((i, j))
                        if blk is not None:
                            ops.halfdiff_dot(blk.bufs["pAx_A"], blk.bufs["pPr_A"], row.dy,
                                             self.slot[("cross", (i, j))])

    def _kkt_collect(self, vals, restarts: bool):
        """Report and per-block table of a pass from its reduction slots."""
        local = {}
        for (i, j) in self.comm.local:
            r = np.zeros(NFIELDS)
            kr = vals[self.slot[("kkt_rows", i)]]
            kc = vals[self.slot[("kkt_cols", j)]]
            r[F_RP2] = kr[0]
            r[F_PEN] = float("inf") if kr[3] > 0 else kr[1] - kr[2]
            r[F_RD2], r[F_CX], r[F_RCX], r[F_DX2] = kc[0], kc[1], kc[2], kc[3]
            if restarts:
                pr = vals[self.slot[("probe", i)]]
                r[F_DY2] = pr[0]
                r[F_CROSS] = pr[1] if self.C == 1 else vals[self.slot[("cross", (i, j))], 0]
            r[F_TIME] = time.monotonic() - self._started if (i, j) == (0, 0) else 0.0
            local[(i, j)] = r
        tab = self._table(local)
        rp_sq = self._axis_sum(tab, F_RP2, "R")
        rd_sq = self._axis_sum(tab, F_RD2, "C")
        obj_p = self._axis_sum(tab, F_CX, "C")
        pen = self._axis_sum(tab, F_PEN, "R")
        cdot = self._axis_sum(tab, F_RCX, "C")
        obj_d = -pen + cdot
        rep = Report(
            r_primal=math.sqrt(rp_sq) / (1.0 + self.bnorm),
            r_dual=math.sqrt(rd_sq) / (1.0 + self.cnorm),
            r_gap=gap_residual(obj_p, obj_d),
            obj_primal=obj_p + self.const,
            obj_dual=obj_d + self.const,
        )
        # evaluate_kkt ledger: C vec + R scalar, R vec + C scalar x2 + R scalar + C scalar
        self.ledger.vec("C", "m")
        self.ledger.vec("R", "n")
        self.ledger.scalar("R", 2)
        self.ledger.scalar("C", 3)
        return rep, tab

    def _anchor_distances(self):
        ops = self.ops
        for j, col in self.cols.items():
            ops.anchor(col.x, col.x0, self.slot[("anchor_x", j)])
        for i, row in self.rows.items():
            ops.anchor(row.y, row.y0, self.slot[("anchor_y", i)])
        vals = ops.read_slots(self.nslots)
        local = {(i, j): np.array([vals[self.slot[("anchor_x", j)], 0], vals[self.slot[("anchor_y", i)], 0]])
                 for (i, j) in self.comm.local}
        tab = self._table(local)
        self.ledger.scalar("G", 2)
        return self._g_sum(tab, 0, self.R), self._g_sum(tab, 1, self.C)

    def _snapshot_xy(self):
        self._sync_shards()
        xs = {j: self._from_internal_col(j, c.x.detach()).copy() for j, c in self.cols.items()}
        ys = {i: self._from_internal_row(i, r.y.detach()).copy() for i, r in self.rows.items()}
        return xs, ys

    # The loop of iterate_epoch (pdhg_engine.py:364-476), split so a caller
    # (bench.py) can time individual passes: start() -> step()* -> finish().
    def start(self, eta: float, omega: float, trace=None, log_hook=None):
        o = self.opts
        for col in self.cols.values():
            self.ops.init_primal(col)
            col.xbar.zero_()
        for row in self.rows.values():
            row.y.zero_()
            row.y0.zero_()
        self._pid = Pid(o.pid_kp, o.pid_ki, o.pid_kd)
        self._s = dict(eta=eta, omega=omega, base_fp=None, prev_fp=None, inner_k=0, epoch=0, total=0,
                       status=None, report=None, report_at=-1, trace=trace, log_hook=log_hook,
                       keep=getattr(trace, "keep", None) if trace is not None else None)
        self._started = time.monotonic()
        self._t_loop = time.perf_counter()

    def step(self, device_loop: bool = False) -> bool:
        """Iterations up to the next KKT pass, then the pass. True when the
        loop terminated (status set). device_loop: run as many KKT intervals
        as the device-side loop decides to (run() does; bench.py times single
        intervals)."""
        o, ops, st = self.opts, self.ops, self._s
        K = o.kkt_interval
        if st["total"] >= o.max_iterations:
            st["status"] = ITERATION_LIMIT
            return True
        if device_loop and st["total"] % K == 0 and st["total"] + K <= o.max_iterations and self._loop_ok():
            return self._step_device_loop()
        eta, omega = st["eta"], st["omega"]
        tau, sigma = eta / omega, eta * omega
        total = st["total"]
        target = min((total // K + 1) * K, o.max_iterations)
        # the device step struct already holds (tau, sigma, gamma) and the
        # advanced Halpern counter unless a restart changed them: skip the
        # H2D write then (launch-bound LPs pay it once per pass otherwise)
        key = (tau, sigma, o.gamma, st["inner_k"])
        if key != st.get("device_step"):
            ops.set_step(tau, sigma, o.gamma, st["inner_k"])
        self.count_iterations(target - total)
        trace = st["trace"]
        if trace is None:
            if target % K == 0 and self.opts.cluster_fused_pass and self._cluster():
                # the KKT pass that follows is computed inside the same cluster launch
                self._fuse_pass_mode = 2 if o.restarts else 1
            with nvtx_range("gridlp.iterations"):
                self._run_iterations(target - total)
            st["inner_k"] += target - total
            total = target
            st["device_step"] = (tau, sigma, o.gamma, st["inner_k"])
        else:
            while total < target:
                self._launch_iterations(1)
                total += 1
                st["inner_k"] += 1
                if st["keep"] is None or total in st["keep"]:
                    xs, ys = self._snapshot_xy()
                    trace.append((total, np.concatenate([xs[j] for j in sorted(xs)]),
                                  np.concatenate([ys[i] for i in sorted(ys)])))
        st["total"] = total
        if total % K != 0:
            return False
        with nvtx_range("gridlp.kkt_pass"):
            report, tab = self._kkt(tau, o.restarts)
        return self._post_pass(report, tab, total, eta, omega)

    def _post_pass(self, report, tab, total: int, eta: float, omega: float) -> bool:
        """The host logic after a KKT pass (pdhg_engine.py:402-476):
        log, termination, restart decision and PID update. True when the
        loop terminated."""
        o, st = self.opts, self._s
        self.passes += 1
        st["report"], st["report_at"] = report, total
        if st["log_hook"] is not None:
            st["log_hook"](total, report, omega, eta, st["epoch"])
        if _broken(report):
            st["status"] = NUMERICAL_FAILURE
            return True
        if report.overall <= o.tolerance:
            st["status"] = OPTIMAL
            return True
        if o.restarts:
            self.ledger.vec("C", "m")
            self.ledger.scalar("G", 3)
            dx_sq = self._g_sum(tab, F_DX2, self.R)
            dy_sq = self._g_sum(tab, F_DY2, self.C)
            cross = self._g_sum(tab, F_CROSS)
            value = (omega / eta) * dx_sq + dy_sq / (eta * omega) + 2.0 * cross
            fp = math.sqrt(max(value, 0.0))
            if st["base_fp"] is None:
                st["base_fp"] = fp
            if restart_decision(st["base_fp"], fp, st["prev_fp"], st["inner_k"], total,
                                o.beta_sufficient, o.beta_necessary, o.beta_artificial):
                d_x_sq, d_y_sq = self._anchor_distances()
                st["omega"] = self._pid.update(math.sqrt(d_x_sq), math.sqrt(d_y_sq), omega,
                                               o.omega_min, o.omega_max)
                st["inner_k"] = 0
                st["epoch"] += 1
                st["base_fp"] = fp
                st["prev_fp"] = None
            else:
                st["prev_fp"] = fp
        if o.time_limit_seconds is not None:
            self.ledger.scalar("G")
            if self._g_sum(tab, F_TIME) >= o.time_limit_seconds:
                st["status"] = TIME_LIMIT
                return True
        return False

    # ------------------------------------------------ device-side loop
    def _loop_ok(self) -> bool:
        o, st = self.opts, self._s
        want = self._cluster() if o.device_loop is None else o.device_loop
        return (want and not getattr(self, "_loop_off", False) and self.comm.kind == "virtual"
                and self.R == 1 and self.C == 1 and not self._banded and o.use_graphs
                and hasattr(self.ops, "loop_graph") and o.time_limit_seconds is None and st["trace"] is None
                and self.iteration_events is None and not self._persistent() and self.device.type == "cuda")

    def _loop_build(self):
        o, ops = self.opts, self.ops
        K = o.kkt_interval
        cap = max(1, int(o.device_loop_passes))
        self._loop_cap = cap
        self._loop_dev = torch.zeros(ctypes.sizeof(native.Loop), dtype=torch.uint8, device=self.device)
        self._ring_dev = torch.zeros((cap, native.LOOP_REC), dtype=torch.float64, device=self.device)
        (i, _), = self.rows.items()
        (j, _), = self.cols.items()
        self._loop_slots = (self.slot[("kkt_rows", i)], self.slot[("kkt_cols", j)],
                            self.slot[("probe", i)] if o.restarts else self.slot[("kkt_rows", i)])

        def interval():
            if self.opts.cluster_fused_pass and self._cluster():
                self._fuse_pass_mode = 2 if o.restarts else 1
            self._launch_iterations(K)
            self._kkt_launch(o.restarts)

        cur = torch.cuda.current_stream(self.device)
        ts = torch.cuda.Stream(self.device)
        ts.wait_stream(cur)
        with torch.cuda.stream(ts):
            self._loop_graph = ops.loop_graph(interval, self._loop_dev, self._ring_dev)
        cur.wait_stream(ts)

    def _step_device_loop(self) -> bool:
        """KKT intervals on the device until a pass terminates, restarts or
        reaches a limit (one graph launch), then the host replays every
        pass's bookkeeping in order — the same code as step() — and checks
        that its decisions are the device's."""
        o, ops, st = self.opts, self.ops, self._s
        K = o.kkt_interval
        eta, omega = st["eta"], st["omega"]
        tau, sigma = eta / omega, eta * omega
        key = (tau, sigma, o.gamma, st["inner_k"])
        if key != st.get("device_step"):
            ops.set_step(tau, sigma, o.gamma, st["inner_k"])
        if getattr(self, "_loop_graph", None) is None:
            try:
                self._loop_build()
            except native.GridlpError as exc:
                log.warning("device-side loop unavailable (%s); host-driven intervals", exc)
                self._loop_off = True
                return self.step()
        L = native.Loop()
        L.eta, L.omega, L.bnorm, L.cnorm = eta, omega, self.bnorm, self.cnorm
        L.obj_const, L.tolerance = self.const, o.tolerance
        L.beta_sufficient, L.beta_necessary, L.beta_artificial = o.beta_sufficient, o.beta_necessary, o.beta_artificial
        L.has_base = int(st["base_fp"] is not None)
        L.base_fp = st["base_fp"] if st["base_fp"] is not None else 0.0
        L.has_prev = int(st["prev_fp"] is not None)
        L.prev_fp = st["prev_fp"] if st["prev_fp"] is not None else 0.0
        L.total, L.inner_k, L.max_iterations, L.kkt_interval = st["total"], st["inner_k"], o.max_iterations, K
        budget = getattr(self, "loop_budget", None)      # bench.py: exactly its timed passes
        cap = self._loop_cap if budget is None else max(1, min(self._loop_cap, int(budget)))
        L.max_passes, L.restarts = cap, int(o.restarts)
        L.slot_rows, L.slot_cols, L.slot_probe = self._loop_slots
        L.passes, L.stopped = 0, 0
        self._loop_dev.copy_(torch.frombuffer(bytearray(L), dtype=torch.uint8))
        with nvtx_range("gridlp.device_loop"):
            self._loop_graph.replay()
            out = native.Loop.from_buffer_copy(self._loop_dev.cpu().numpy().tobytes())
        n = int(out.passes)
        ring = self._ring_dev[:n].cpu().numpy()
        ops.launches += self._loop_graph.launches * (n - 1)
        vals = np.zeros((self.nslots, native.MAX_RED))
        sr, sc, sp = self._loop_slots
        done = False
        for p in range(n):
            rec = ring[p]
            self.count_iterations(K)
            st["inner_k"] += K
            st["total"] += K
            st["device_step"] = (tau, sigma, o.gamma, st["inner_k"])
            vals[sr, :4] = rec[0:4]
            vals[sc, :4] = rec[4:8]
            if o.restarts:
                vals[sp, :2] = rec[8:10]
            epoch = st["epoch"]
            report, tab = self._kkt_collect(vals, o.restarts)
            done = self._post_pass(report, tab, st["total"], eta, omega)
            host_stop = done or st["epoch"] != epoch
            dev_stop = rec[11] != 0.0
            limit = st["total"] + K > o.max_iterations or p + 1 >= cap
            if (p < n - 1 and (host_stop or dev_stop)) or (p == n - 1 and (not dev_stop or (not host_stop and not limit))):
                raise RuntimeError(f"device-side loop diverged from the host decision at pass {p} of {n} "
                                   f"(iteration {st['total']})")
        return done

    def finish(self):
        o, ops, st = self.opts, self.ops, self._s
        eta, omega = st["eta"], st["omega"]
        report, status = st["report"], st["status"]
        if st["report_at"] != st["total"]:
            ops.set_step(eta / omega, eta * omega, o.gamma, st["inner_k"])
            report, _ = self._kkt(eta / omega, False)
            if status != NUMERICAL_FAILURE and _broken(report):
                status = NUMERICAL_FAILURE
        self._sync_shards()
        if self.device.type == "cuda":
            torch.cuda.synchronize(self.device)
        self.timings["main_loop_s"] = time.perf_counter() - self._t_loop
        return {"status": status, "report": report, "iterations": st["total"],
                "restarts": st["epoch"], "omega": omega, "eta": eta}

    def run(self, eta: float, omega: float, trace=None, log_hook=None):
        """iterate_epoch (pdhg_engine.py:364-476). Returns a dict outcome."""
        self.start(eta, omega, trace, log_hook)
        while not self.step(device_loop=True):
            pass
        return self.finish()

    def count_iterations(self, n: int):
        self.ledger.vec("R", "n", n)
        self.ledger.vec("C", "m", n)

    def solution_original(self):
        """(x, y) as host arrays in the user's index order, by one device
        scatter each through the composed (layout permutation, internal
        order) index of the device setup; None when that index is not
        available (host setup, band problems, one block per process)."""
        if self.comm.kind != "virtual" or len(self._col_idx) != self.C or len(self._row_idx) != self.R:
            return None
        x = torch.empty(self.layout.num_cols, dtype=torch.float64, device=self.device)
        y = torch.empty(self.layout.num_rows, dtype=torch.float64, device=self.device)
        for j, idx in self._col_idx.items():
            x[idx] = self.cols[j].x
        for i, idx in self._row_idx.items():
            y[idx] = self.rows[i].y
        return x.cpu().numpy(), y.cpu().numpy()

    def solution_blocks(self):
        """x blocks of grid columns (from devices (0, j)) and y blocks of grid
        rows (from (i, 0)) as host arrays (solver_driver.py:246-248)."""
        if self.comm.kind == "virtual":
            xs = [self._from_internal_col(j, self.cols[j].x) for j in range(self.C)]
            ys = [self._from_internal_row(i, self.rows[i].y) for i in range(self.R)]
            return xs, ys
        lay = self.layout
        lengths = {(i, j): max(int(lay.col_cuts[j + 1] - lay.col_cuts[j]), int(lay.row_cuts[i + 1] - lay.row_cuts[i]))
                   for i in range(self.R) for j in range(self.C)}
        xl = {c: self.cols[c[1]].x for c in self.comm.local}
        yl = {c: self.rows[c[0]].y for c in self.comm.local}
        xlen = {(i, j): int(lay.col_cuts[j + 1] - lay.col_cuts[j]) for i in range(self.R) for j in range(self.C)}
        ylen = {(i, j): int(lay.row_cuts[i + 1] - lay.row_cuts[i]) for i in range(self.R) for j in range(self.C)}
        del lengths
        xa = self.comm.gather_vectors(xl, xlen, self.device)
        ya = self.comm.gather_vectors(yl, ylen, self.device)
        xs = [self._from_internal_col(j, xa[(0, j)]) for j in range(self.C)]
        ys = [self._from_internal_row(i, ya[(i, 0)]) for i in range(self.R)]
        return xs, ys
