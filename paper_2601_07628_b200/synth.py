"""Device generators for the large BASELINE configs.

The reference's generators.py has no power-law or multi-commodity-flow kind
(generators.py:23), and at 200M-500M nonzeros a numpy build would dominate
the run, so these instances are generated on the GPU through the C ABI
(csrc/gridlp_gen.cu). Every random number is a counter-based hash of
(seed, stream, global index), so an instance is independent of grid, launch
shape and device; oracle/synth_oracle.py restates both generators in numpy
and tests/test_gpu_synth.py checks the device output against it bit for bit
at small sizes.

* `PowerLawSpec` (cfg3): Chung-Lu-style rows. Row r draws
  d_r = clip(floor(nnz_target * w_r / sum(w) + u_r), 1, n) columns with
  w_r = (r + 1)^-alpha (heavy rows first, the natural order the paper's
  shuffle is meant to break); each draw is c = floor((1 + u kappa)^5) - 1,
  a power law of exponent 0.8 over columns (heavy columns first); duplicate
  draws collapse, so the realised nnz is a little below the target. Values
  U[-1, 1); the LP is the reference generator's feasible wrapper
  (generators.py:120-142): box [box_low, box_high], rhs = A x_hat with
  x_hat ~ U[1, 3), a fraction of rows ranged by U[0.1, 1) on each side,
  c ~ U[-1, 1).
* `McfSpec` (cfg4): block-angular multi-commodity flow. A random directed
  graph (V nodes, E arcs, no self-loops) and K commodities; variable k*E + e
  is commodity k's flow on arc e. Rows k*V + v are flow conservation
  (+1 out-arcs, -1 in-arcs) with lo = hi = the divergence of a planted flow
  x_hat ~ U[0.5, 1.5); rows K*V + e couple the commodities on arc e,
  sum_k x_ke <= 1.25 * (planted load). Costs U[1, 10), box [0, 4].
* `PlantedSpec` (cfg5): a uniform random matrix (d column draws per row)
  with a planted primal-dual optimum (x*, y*): x* puts 30 % of the
  variables at the lower and 10 % at the upper bound, y* makes 35 % of the
  rows active at their lower and 35 % at their upper bound, the objective is
  c = Aᵀ y* + r* with a reduced cost r* complementary to x*. (x*, y*)
  satisfies the KKT conditions exactly, so the optimal objective is c·x* —
  an analytic oracle that needs no CPU solve, for instances too large for
  one GPU or the host.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import native
from .problem import LpProblem, SparseMatrix

HASH_MUL = np.uint64(0x100000001B3)


def _mix(z: np.ndarray) -> np.ndarray:
    z = z + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def host_u01(seed: int, stream: int, a, b=0) -> np.ndarray:
    """u(seed, stream, a, b) of include/gridlp_b200.h on the host (small
    host-side draws: row allocations, the MCF graph)."""
    with np.errstate(over="ignore"):
        s = _mix(np.uint64(seed) * HASH_MUL + np.uint64(stream))
        h = _mix(_mix(s ^ np.asarray(a, dtype=np.uint64)) ^ np.asarray(b, dtype=np.uint64))
    return (h >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


@dataclass(frozen=True)
class PowerLawSpec:
    num_rows: int
    num_cols: int
    nnz_target: int
    alpha: float = 0.8
    inequality_fraction: float = 0.3
    box_low: float = 0.0
    box_high: float = 4.0
    seed: int = 0

    def __post_init__(self):
        if self.num_rows < 1 or self.num_cols < 1 or self.nnz_target < self.num_rows:
            raise ValueError("need num_rows, num_cols >= 1 and nnz_target >= num_rows")
        if self.num_cols >= 2 ** 31 - 1 or self.num_rows >= 2 ** 31 - 1:
            raise ValueError("rows and columns must be < 2^31")
        if not 0.0 <= self.inequality_fraction <= 1.0:
            raise ValueError("inequality_fraction must be in [0, 1]")
        if self.box_low >= self.box_high:
            raise ValueError("box_low must be below box_high")


@dataclass(frozen=True)
class McfSpec:
    num_nodes: int
    num_arcs: int
    num_commodities: int
    capacity_factor: float = 1.25
    seed: int = 0

    def __post_init__(self):
        if self.num_nodes < 2 or self.num_arcs < 1 or self.num_commodities < 1:
            raise ValueError("need >= 2 nodes, >= 1 arc, >= 1 commodity")
        if self.num_commodities * self.num_arcs >= 2 ** 31 - 1:
            raise ValueError("K * E must be < 2^31 (int32 column indices)")


@dataclass(frozen=True)
class PlantedSpec:
    num_rows: int
    num_cols: int
    draws_per_row: int = 8
    box_low: float = 0.0
    box_high: float = 4.0
    seed: int = 0

    def __post_init__(self):
        if self.num_rows < 1 or self.num_cols < 1 or self.draws_per_row < 1:
            raise ValueError("need num_rows, num_cols, draws_per_row >= 1")
        if self.num_cols >= 2 ** 31 - 1 or self.num_rows * self.draws_per_row >= 2 ** 31:
            raise ValueError("one-piece generation needs < 2^31 columns and draws")
        if self.box_low >= self.box_high:
            raise ValueError("box_low must be below box_high")


def powerlaw_row_alloc(spec: PowerLawSpec) -> np.ndarray:
    """Column draws per row (host numpy, shared formula with the oracle)."""
    m, n = spec.num_rows, spec.num_cols
    w = (np.arange(m, dtype=np.float64) + 1.0) ** -spec.alpha
    expected = float(spec.nnz_target) * (w / w.sum())
    d = np.floor(expected + host_u01(spec.seed, 0, np.arange(m))).astype(np.int64)
    return np.clip(d, 1, n)


def powerlaw_kappa(n: int) -> float:
    return (n + 1.0) ** 0.2 - 1.0


def mcf_graph(spec: McfSpec):
    """Arcs (tail, head) and the node adjacency (CSR over nodes, arcs
    ascending, sign +1 out / -1 in)."""
    V, E, s = spec.num_nodes, spec.num_arcs, spec.seed
    e = np.arange(E)
    tail = np.floor(host_u01(s, 10, e) * V).astype(np.int64)
    off = 1 + np.floor(host_u01(s, 11, e) * (V - 1)).astype(np.int64)
    head = (tail + off) % V
    node = np.concatenate([tail, head])
    arc = np.concatenate([e, e])
    sign = np.concatenate([np.ones(E, np.int8), -np.ones(E, np.int8)])
    order = np.lexsort((arc, node))
    adj_ptr = np.concatenate([[0], np.cumsum(np.bincount(node, minlength=V))]).astype(np.int32)
    return tail, head, adj_ptr, arc[order].astype(np.int32), sign[order]


class _Gen:
    def __init__(self, device):
        self.lib = native.load()
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())

    def stream(self):
        return torch.cuda.current_stream(self.device).cuda_stream

    def ws(self, items, rows):
        nb = int(self.lib._lib.gridlp_gen_workspace_bytes(int(items), int(rows)))
        return torch.empty(nb, dtype=torch.uint8, device=self.device), nb

    def scan(self, lens: torch.Tensor) -> torch.Tensor:
        out = torch.empty_like(lens)
        ws, nb = self.ws(1, lens.numel())
        self.lib.call("gridlp_gen_scan64", lens.data_ptr(), out.data_ptr(), lens.numel(), ws.data_ptr(), nb,
                      self.stream())
        return out

    def uniform(self, seed, stream_id, n, lo, hi) -> torch.Tensor:
        out = torch.empty(max(n, 1), dtype=torch.float64, device=self.device)[:n]
        self.lib.call("gridlp_gen_uniform", seed, stream_id, 0, n, float(lo), float(hi),
                      out.data_ptr() if n else None, self.stream())
        return out

    def spmv_seq(self, ptr, cols, vals, m, x) -> torch.Tensor:
        y = torch.empty(max(m, 1), dtype=torch.float64, device=self.device)[:m]
        self.lib.call("gridlp_csr_spmv_seq", ptr.data_ptr(), cols.data_ptr(), vals.data_ptr(), m, x.data_ptr(),
                      y.data_ptr() if m else None, self.stream())
        return y


@dataclass
class DeviceLp:
    """A generated LP resident on the device (int64 row pointers, int32
    columns, FP64 values and vectors)."""

    num_rows: int
    num_cols: int
    row_ptr: torch.Tensor
    cols: torch.Tensor
    vals: torch.Tensor
    objective: torch.Tensor
    var_lower: torch.Tensor
    var_upper: torch.Tensor
    con_lower: torch.Tensor
    con_upper: torch.Tensor
    x_hat: torch.Tensor

    @property
    def nnz(self) -> int:
        return int(self.cols.numel())

    def to_problem(self, name: str = "synthetic") -> LpProblem:
        """Host LpProblem (the public solve() input); no validation pass."""
        c = lambda t: t.cpu().numpy()  # noqa: E731
        A = SparseMatrix(self.num_rows, self.num_cols, c(self.row_ptr), c(self.cols).astype(np.int64), c(self.vals),
                         check=False)
        return LpProblem(A, c(self.objective), c(self.var_lower), c(self.var_upper), c(self.con_lower),
                         c(self.con_upper), name=name)


def generate_powerlaw(spec: PowerLawSpec, device=None) -> DeviceLp:
    g = _Gen(device)
    dev, m, n, seed = g.device, spec.num_rows, spec.num_cols, spec.seed
    alloc = powerlaw_row_alloc(spec)
    total = int(alloc.sum())
    if total >= 2 ** 31:
        raise ValueError("power-law draws must be < 2^31 per instance (per-call sort limit)")
    lens = torch.zeros(m + 1, dtype=torch.int64, device=dev)
    lens[:m] = torch.from_numpy(alloc).to(dev)
    alloc_ptr = g.scan(lens)
    del lens
    raw = torch.empty(total, dtype=torch.int32, device=dev)
    g.lib.call("gridlp_gen_powerlaw_sample", seed, alloc_ptr.data_ptr(), m, n, powerlaw_kappa(n), raw.data_ptr(),
               g.stream())
    srt = torch.empty_like(raw)
    ws, nb = g.ws(total, m)
    g.lib.call("gridlp_gen_sort_rows", alloc_ptr.data_ptr(), m, total, raw.data_ptr(), srt.data_ptr(), ws.data_ptr(),
               nb, g.stream())
    del raw, ws
    counts = torch.empty(m + 1, dtype=torch.int64, device=dev)
    g.lib.call("gridlp_gen_dedupe_count", alloc_ptr.data_ptr(), srt.data_ptr(), m, 0, n, counts.data_ptr(), g.stream())
    row_ptr = g.scan(counts)
    del counts
    nnz = int(row_ptr[m])
    cols = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)[:nnz]
    vals = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)[:nnz]
    g.lib.call("gridlp_gen_dedupe_fill", alloc_ptr.data_ptr(), srt.data_ptr(), m, 0, 0, n, row_ptr.data_ptr(), seed,
               cols.data_ptr(), vals.data_ptr(), g.stream())
    del srt, alloc_ptr
    x_hat = g.uniform(seed, 3, n, 1.0, 3.0)
    obj = g.uniform(seed, 4, n, -1.0, 1.0)
    b = g.spmv_seq(row_ptr, cols, vals, m, x_hat)
    lo = torch.empty(m, dtype=torch.float64, device=dev)
    hi = torch.empty(m, dtype=torch.float64, device=dev)
    g.lib.call("gridlp_gen_row_bounds", seed, m, float(spec.inequality_fraction), b.data_ptr(), lo.data_ptr(),
               hi.data_ptr(), g.stream())
    f64 = dict(dtype=torch.float64, device=dev)
    return DeviceLp(m, n, row_ptr, cols, vals, obj, torch.full((n,), spec.box_low, **f64),
                    torch.full((n,), spec.box_high, **f64), lo, hi, x_hat)


def generate_mcf(spec: McfSpec, device=None) -> DeviceLp:
    g = _Gen(device)
    dev, seed = g.device, spec.seed
    K, V, E = spec.num_commodities, spec.num_nodes, spec.num_arcs
    m, n = K * V + E, K * E
    _, _, adj_ptr, adj_arc, adj_sign = mcf_graph(spec)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    d_ptr, d_arc, d_sign = t(adj_ptr), t(adj_arc), t(adj_sign)
    lens = torch.empty(m + 1, dtype=torch.int64, device=dev)
    g.lib.call("gridlp_gen_mcf_row_lengths", K, V, E, d_ptr.data_ptr(), lens.data_ptr(), g.stream())
    row_ptr = g.scan(lens)
    del lens
    nnz = int(row_ptr[m])
    cols = torch.empty(nnz, dtype=torch.int32, device=dev)
    vals = torch.empty(nnz, dtype=torch.float64, device=dev)
    g.lib.call("gridlp_gen_mcf_fill", K, V, E, d_ptr.data_ptr(), d_arc.data_ptr(), d_sign.data_ptr(),
               row_ptr.data_ptr(), cols.data_ptr(), vals.data_ptr(), g.stream())
    x_hat = g.uniform(seed, 12, n, 0.5, 1.5)
    obj = g.uniform(seed, 13, n, 1.0, 10.0)
    b = g.spmv_seq(row_ptr, cols, vals, m, x_hat)
    lo = b.clone()
    hi = b.clone()
    lo[K * V:] = -float("inf")
    hi[K * V:] = b[K * V:] * float(spec.capacity_factor)
    f64 = dict(dtype=torch.float64, device=dev)
    return DeviceLp(m, n, row_ptr, cols, vals, obj, torch.zeros(n, **f64), torch.full((n,), 4.0, **f64), lo, hi,
                    x_hat)


@dataclass
class PlantedLp(DeviceLp):
    y_star: torch.Tensor = None

    def optimal_objective(self) -> float:
        """c·x* — the planted optimum (sequential host sum of the device arrays)."""
        return float(np.dot(self.objective.cpu().numpy(), self.x_hat.cpu().numpy()))


class PlantedBands:
    """The cfg5 planted LP generated band by band: `block(r0, r1, c0, c1)`
    builds one grid block, `row_data` / `col_data` one row / column band's
    vectors, and no device ever holds more than one block plus a chunk of
    draws — the path for LPs whose A + Aᵀ exceed one GPU. Every value is the
    one-piece instance's bit for bit: b = A x* is summed over each full row
    (regenerated from the hash), c = Aᵀ y* + r* is accumulated column by
    column over all rows in ascending order, chunk after chunk."""

    def __init__(self, spec: PlantedSpec, device=None, chunk_draws: int = 1 << 27):
        self.spec = spec
        self.g = _Gen(device)
        self.chunk_rows = max(1, chunk_draws // spec.draws_per_row)
        self.f64 = dict(dtype=torch.float64, device=self.g.device)

    @property
    def shape(self):
        return self.spec.num_rows, self.spec.num_cols

    def _sorted_rows(self, r0: int, r1: int):
        """Draws of rows [r0, r1), sorted inside each row."""
        g, sp_, d = self.g, self.spec, self.spec.draws_per_row
        m = r1 - r0
        raw = torch.empty(max(m * d, 1), dtype=torch.int32, device=g.device)
        g.lib.call("gridlp_gen_band_draws", sp_.seed, r0, m, d, sp_.num_cols, raw.data_ptr(), g.stream())
        ptr = torch.arange(m + 1, dtype=torch.int64, device=g.device) * d
        srt = torch.empty_like(raw)
        ws, nb = g.ws(m * d, m)
        g.lib.call("gridlp_gen_sort_rows", ptr.data_ptr(), m, m * d, raw.data_ptr(), srt.data_ptr(), ws.data_ptr(), nb,
                   g.stream())
        return ptr, srt

    def _band_csr(self, ptr, srt, m: int, r0: int, c0: int, c1: int):
        """Distinct entries of the sorted rows inside [c0, c1): int64 row
        pointers, local int32 columns, values."""
        g = self.g
        counts = torch.empty(m + 1, dtype=torch.int64, device=g.device)
        g.lib.call("gridlp_gen_dedupe_count", ptr.data_ptr(), srt.data_ptr(), m, c0, c1, counts.data_ptr(), g.stream())
        out_ptr = g.scan(counts)
        nnz = int(out_ptr[m])
        cols = torch.empty(nnz + 8, dtype=torch.int32, device=g.device)
        vals = torch.empty(nnz + 8, **self.f64)
        g.lib.call("gridlp_gen_dedupe_fill", ptr.data_ptr(), srt.data_ptr(), m, r0, c0, c1, out_ptr.data_ptr(),
                   self.spec.seed, cols.data_ptr(), vals.data_ptr(), g.stream())
        return out_ptr, cols, vals, nnz

    def _chunks(self, r0: int, r1: int):
        for a in range(r0, r1, self.chunk_rows):
            yield a, min(r1, a + self.chunk_rows)

    def block(self, r0: int, r1: int, c0: int, c1: int):
        """Grid block rows [r0, r1) x columns [c0, c1) as DeviceCsrArrays
        (int32 row pointers, local column ids, entries sorted by column)."""
        from .blocks import DeviceCsrArrays

        parts = []
        for a, b in self._chunks(r0, r1):
            ptr, srt = self._sorted_rows(a, b)
            parts.append(self._band_csr(ptr, srt, b - a, a, c0, c1))
            del ptr, srt
        nnz = sum(p[3] for p in parts)
        if nnz >= 2 ** 31 - 64:
            raise ValueError("block nnz must be < 2^31: use a finer grid")
        dev = self.g.device
        rp = torch.empty(r1 - r0 + 1, dtype=torch.int64, device=dev)
        cols = torch.empty(nnz + 8, dtype=torch.int32, device=dev)
        vals = torch.empty(nnz + 8, **self.f64)
        rp[0], row, off = 0, 0, 0
        for p_, c_, v_, k in parts:
            mm = p_.numel() - 1
            rp[row + 1: row + mm + 1] = p_[1:] + off
            cols[off: off + k] = c_[:k]
            vals[off: off + k] = v_[:k]
            row, off = row + mm, off + k
        return DeviceCsrArrays(r1 - r0, c1 - c0, nnz, rp.to(torch.int32), cols, vals)

    def row_data(self, r0: int, r1: int):
        """(con_lower, con_upper, y*) of rows [r0, r1); b = A x* over full rows."""
        g, sp_ = self.g, self.spec
        m = r1 - r0
        b = torch.empty(max(m, 1), **self.f64)[:m]
        for a, e in self._chunks(r0, r1):
            ptr, srt = self._sorted_rows(a, e)
            g.lib.call("gridlp_gen_planted_row_dot", ptr.data_ptr(), srt.data_ptr(), e - a, a, sp_.seed, sp_.box_low,
                       sp_.box_high, b[a - r0:].data_ptr(), g.stream())
        y, lo, hi = (torch.empty(max(m, 1), **self.f64)[:m] for _ in range(3))
        if m:
            g.lib.call("gridlp_gen_planted_rows", sp_.seed, r0, m, b.data_ptr(), y.data_ptr(), lo.data_ptr(),
                       hi.data_ptr(), g.stream())
        return lo, hi, y

    def col_data(self, c0: int, c1: int):
        """(c, var_lower, var_upper, x*) of columns [c0, c1); c = Aᵀ y* + r*
        accumulated over every row chunk in ascending order."""
        g, sp_ = self.g, self.spec
        n = c1 - c0
        acc = torch.zeros(max(n, 1), **self.f64)[:n]
        wsb = 0
        for a, e in self._chunks(0, sp_.num_rows):
            ptr, srt = self._sorted_rows(a, e)
            bp, bc, bv, nnz = self._band_csr(ptr, srt, e - a, a, c0, c1)
            del ptr, srt
            need = int(g.lib._lib.gridlp_setup_workspace_bytes(nnz + 64, max(e - a, n) + 64))
            if need > wsb:
                ws, wsb = torch.empty(need, dtype=torch.uint8, device=g.device), need
            tptr = torch.empty(n + 1, dtype=torch.int32, device=g.device)
            trow = torch.empty(nnz + 8, dtype=torch.int32, device=g.device)
            tval = torch.empty(nnz + 8, **self.f64)
            g.lib.call("gridlp_csr_transpose", bp.to(torch.int32).data_ptr(), bc.data_ptr(), bv.data_ptr(), e - a, n,
                       nnz, tptr.data_ptr(), trow.data_ptr(), tval.data_ptr(), ws.data_ptr(), wsb, g.stream())
            g.lib.call("gridlp_gen_col_accumulate", tptr.data_ptr(), trow.data_ptr(), tval.data_ptr(), n, a, sp_.seed,
                       acc.data_ptr(), g.stream())
        x, r = torch.empty(max(n, 1), **self.f64)[:n], torch.empty(max(n, 1), **self.f64)[:n]
        c = torch.empty(max(n, 1), **self.f64)[:n]
        if n:
            g.lib.call("gridlp_gen_planted_cols", sp_.seed, c0, n, sp_.box_low, sp_.box_high, x.data_ptr(), r.data_ptr(),
                       g.stream())
            g.lib.call("gridlp_gen_add", acc.data_ptr(), r.data_ptr(), n, c.data_ptr(), g.stream())
        return c, torch.full((n,), sp_.box_low, **self.f64), torch.full((n,), sp_.box_high, **self.f64), x


def generate_planted(spec: PlantedSpec, device=None) -> PlantedLp:
    """The whole cfg5 instance on one device (small sizes; `PlantedBands`
    builds the same instance block by block)."""
    bands = PlantedBands(spec, device)
    m, n = spec.num_rows, spec.num_cols
    blk = bands.block(0, m, 0, n)
    lo, hi, y = bands.row_data(0, m)
    c, vlo, vhi, x = bands.col_data(0, n)
    return PlantedLp(m, n, blk.ptr.to(torch.int64), blk.col[: blk.nnz], blk.val[: blk.nnz], c, vlo, vhi, lo, hi, x,
                     y_star=y)


class _Shape:
    """Matrix stand-in of a band problem: dimensions only."""

    row_offsets = col_indices = values = None

    def __init__(self, m: int, n: int):
        self.num_rows, self.num_cols = m, n

    @property
    def nnz(self):
        raise ValueError("a band problem has no global matrix; its blocks are generated per device")


class BandProblem:
    """LpProblem stand-in for solve() whose blocks and band vectors come from
    a generator (`bands`) instead of host arrays: each device builds only its
    own block, so the LP can exceed one GPU's memory and the host's. Needs
    permutation "none" and partitioning "uniform" (the generator is already
    unstructured); x / y are returned in full on the host."""

    objective_constant = 0.0
    maximize = False

    def __init__(self, bands: PlantedBands, name: str = "planted"):
        self.bands = bands
        self.matrix = _Shape(*bands.shape)
        self.name = name

    @property
    def num_constraints(self):
        return self.matrix.num_rows

    @property
    def num_variables(self):
        return self.matrix.num_cols
