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
        self.lib.call("gridlp_gen_uniform", seed, stream_id, n, float(lo), float(hi),
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
    g.lib.call("gridlp_gen_dedupe_count", alloc_ptr.data_ptr(), srt.data_ptr(), m, counts.data_ptr(), g.stream())
    row_ptr = g.scan(counts)
    del counts
    nnz = int(row_ptr[m])
    cols = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)[:nnz]
    vals = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)[:nnz]
    g.lib.call("gridlp_gen_dedupe_fill", alloc_ptr.data_ptr(), srt.data_ptr(), m, row_ptr.data_ptr(), seed,
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


def _dedupe_rows(g: _Gen, alloc_ptr, raw, m, seed):
    total = int(raw.numel())
    srt = torch.empty_like(raw)
    ws, nb = g.ws(total, m)
    g.lib.call("gridlp_gen_sort_rows", alloc_ptr.data_ptr(), m, total, raw.data_ptr(), srt.data_ptr(), ws.data_ptr(),
               nb, g.stream())
    del ws
    counts = torch.empty(m + 1, dtype=torch.int64, device=g.device)
    g.lib.call("gridlp_gen_dedupe_count", alloc_ptr.data_ptr(), srt.data_ptr(), m, counts.data_ptr(), g.stream())
    row_ptr = g.scan(counts)
    nnz = int(row_ptr[m])
    cols = torch.empty(max(nnz, 1), dtype=torch.int32, device=g.device)[:nnz]
    vals = torch.empty(max(nnz, 1), dtype=torch.float64, device=g.device)[:nnz]
    g.lib.call("gridlp_gen_dedupe_fill", alloc_ptr.data_ptr(), srt.data_ptr(), m, row_ptr.data_ptr(), seed,
               cols.data_ptr(), vals.data_ptr(), g.stream())
    return row_ptr, cols, vals


def generate_planted(spec: PlantedSpec, device=None) -> PlantedLp:
    g = _Gen(device)
    dev, m, n, seed = g.device, spec.num_rows, spec.num_cols, spec.seed
    f64 = dict(dtype=torch.float64, device=dev)
    lens = torch.full((m + 1,), spec.draws_per_row, dtype=torch.int64, device=dev)
    lens[m] = 0
    alloc_ptr = g.scan(lens)
    raw = torch.empty(m * spec.draws_per_row, dtype=torch.int32, device=dev)
    g.lib.call("gridlp_gen_uniform_sample", seed, alloc_ptr.data_ptr(), m, n, raw.data_ptr(), g.stream())
    row_ptr, cols, vals = _dedupe_rows(g, alloc_ptr, raw, m, seed)
    del raw, alloc_ptr
    x, r = torch.empty(n, **f64), torch.empty(n, **f64)
    g.lib.call("gridlp_gen_planted_cols", seed, n, spec.box_low, spec.box_high, x.data_ptr(), r.data_ptr(), g.stream())
    b = g.spmv_seq(row_ptr, cols, vals, m, x)
    y, lo, hi = torch.empty(m, **f64), torch.empty(m, **f64), torch.empty(m, **f64)
    g.lib.call("gridlp_gen_planted_rows", seed, m, b.data_ptr(), y.data_ptr(), lo.data_ptr(), hi.data_ptr(),
               g.stream())
    # c = Aᵀ y* + r*: sequential sums along the rows of the stored transpose
    nnz = int(cols.numel())
    wsb = int(g.lib._lib.gridlp_setup_workspace_bytes(nnz + 64, max(m, n) + 64))
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    tptr = torch.empty(n + 1, dtype=torch.int32, device=dev)
    tcol = torch.empty(nnz + 8, dtype=torch.int32, device=dev)
    tval = torch.empty(nnz + 8, **f64)
    g.lib.call("gridlp_csr_transpose", row_ptr.to(torch.int32).data_ptr(), cols.data_ptr(), vals.data_ptr(), m, n,
               nnz, tptr.data_ptr(), tcol.data_ptr(), tval.data_ptr(), ws.data_ptr(), wsb, g.stream())
    aty = g.spmv_seq(tptr.to(torch.int64), tcol, tval, n, y)
    del ws, tptr, tcol, tval
    c = torch.empty(n, **f64)
    g.lib.call("gridlp_gen_add", aty.data_ptr(), r.data_ptr(), n, c.data_ptr(), g.stream())
    return PlantedLp(m, n, row_ptr, cols, vals, c, torch.full((n,), spec.box_low, **f64),
                     torch.full((n,), spec.box_high, **f64), lo, hi, x, y_star=y)
