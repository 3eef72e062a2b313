"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

This module is the checker for the B200 path, never part of it. Only
`tests/`, `__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline` leg and
`--impl reference` arm) may import it. The product package
`paper_2601_07628_b200` never imports anything under `oracle/`.

What it is: a numpy restatement of the reference's single-device PDHG oracle
(`reference_solve`, /root/reference/pkg/src/gridlp/solver_driver.py:290-445)
generalised to the lockstep 2D grid the reference simulates
(`solve` + `iterate_epoch`, solver_driver.py:193-272 and
pdhg_engine.py:364-476). All devices of an R x C grid are advanced in one
thread, in lockstep; every axis reduction is summed in ascending device order
exactly like the simulated communicator (comm.py:75-84, :299-303), so a 1x1
grid is bit-identical to `reference_solve` and an R x C grid is
bit-identical to the reference's simulated grid of the same shape.

Arithmetic provenance:
  * sparse products go through scipy's compiled `csr_matvec` (sequential
    left-to-right per row from +0.0, one rounding per multiply and per add) —
    the reference's own third-party kernel (sparse_kernels.py:18-24,
    lp_model.py:98-106; scipy 1.18.1 in this image, `pyproject.toml:12`
    pins only `scipy>=1.10`);
  * norms/dots are numpy `np.dot` (OpenBLAS ddot), as in the reference.

Parity is PINNED: `tests/test_oracle_golden.py` checks this module bit-for-bit
against fixtures produced by importing the reference itself
(`tests/golden/make_golden.py`).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

OPTIMAL = "optimal"
ITER_LIMIT = "iteration_limit"
TIME_LIMIT = "time_limit"
NUM_FAIL = "numerical_failure"


# ---------------------------------------------------------------------------
# matrices (lp_model.py:40-150)
# ---------------------------------------------------------------------------

def csr_from_triplets(m, n, rows, cols, vals) -> sp.csr_matrix:
    """Row-major, column-sorted CSR; duplicates summed in position order
    (follows SparseMatrix.from_coo, lp_model.py:121-141)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    idx = np.lexsort((cols, rows))
    rows, cols, vals = rows[idx], cols[idx], vals[idx]
    if rows.size:
        same = (rows[1:] == rows[:-1]) & (cols[1:] == cols[:-1])
        if same.any():
            run_id = np.concatenate([[0], np.cumsum(~same)])
            vals = np.bincount(run_id, weights=vals)
            first = np.concatenate([[True], ~same])
            rows, cols = rows[first], cols[first]
    ptr = np.zeros(m + 1, dtype=np.int64)
    np.add.at(ptr, rows + 1, 1)
    ptr = np.cumsum(ptr)
    return sp.csr_matrix((vals, cols, ptr), shape=(m, n))


def as_csr(matrix) -> sp.csr_matrix:
    """Accept a reference-style SparseMatrix (row_offsets/col_indices/values)
    or a scipy matrix."""
    if sp.issparse(matrix):
        return sp.csr_matrix(matrix)
    return sp.csr_matrix(
        (np.asarray(matrix.values, dtype=np.float64),
         np.asarray(matrix.col_indices, dtype=np.int64),
         np.asarray(matrix.row_offsets, dtype=np.int64)),
        shape=(int(matrix.num_rows), int(matrix.num_cols)),
    )


def seq_spmv(a: sp.csr_matrix, x: np.ndarray) -> np.ndarray:
    """y = A x through scipy csr_matvec (sparse_kernels.py:18-24)."""
    if x.shape != (a.shape[1],):
        raise ValueError("vector length mismatch")
    return a.dot(x)


def csr_transpose(a: sp.csr_matrix) -> sp.csr_matrix:
    """Explicit transpose with sorted columns (sparse_kernels.py:27-36)."""
    t = a.T.tocsr()
    t.sort_indices()
    return t


# ---------------------------------------------------------------------------
# layout (partition.py:131-337)
# ---------------------------------------------------------------------------

def grid_shape(m: int, n: int, procs: int) -> tuple[int, int]:
    """partition.py:131-150: max usage, then |log(R/C) - log(m/n)|, then
    more rows."""
    want = math.log(max(m, 1) / max(n, 1))
    best_key, best = None, None
    for r in range(1, max(min(procs, m), 1) + 1):
        c = min(procs // r, max(min(procs, n), 1))
        if c < 1:
            continue
        key = (-(r * c), abs(math.log(r / c) - want), -r)
        if best_key is None or key < best_key:
            best_key, best = key, (r, c)
    return best


def shuffle_blocks(length: int, bsize: int, seed: int) -> np.ndarray:
    """partition.py:153-173: Fisher-Yates over ceil(length/bsize) blocks,
    one `rng.integers(0, i+1)` draw per position from the top."""
    if length == 0:
        return np.zeros(0, dtype=np.int64)
    nb = -(-length // bsize)
    order = np.arange(nb, dtype=np.int64)
    gen = np.random.default_rng(seed)
    for i in range(nb - 1, 0, -1):
        k = int(gen.integers(0, i + 1))
        order[i], order[k] = order[k], order[i]
    starts = order * bsize
    lens = np.minimum(starts + bsize, length) - starts
    base = np.repeat(starts - (np.cumsum(lens) - lens), lens)
    return base + np.arange(length, dtype=np.int64)


def even_cuts(length: int, parts: int) -> np.ndarray:
    """partition.py:176-179."""
    return np.array([-(-t * length // parts) for t in range(parts + 1)], dtype=np.int64)


def greedy_cuts(counts: np.ndarray, parts: int) -> np.ndarray:
    """partition.py:182-206, written as the literal sweep."""
    counts = np.asarray(counts)
    n = len(counts)
    if n == 0:
        return np.zeros(parts + 1, dtype=np.int64)
    total = int(counts.sum())
    out, acc, pos = [0], 0, 0
    for p in range(1, parts):
        goal = total * p / parts
        hi = n - (parts - p)
        lo = out[-1] + 1
        while pos < hi and (pos < lo or acc < goal):
            acc += int(counts[pos])
            pos += 1
        out.append(pos)
    out.append(n)
    return np.array(out, dtype=np.int64)


def axis_seeds(seed: int) -> tuple[int, int]:
    """partition.py:257-259."""
    s = np.random.SeedSequence(seed).generate_state(2, dtype=np.uint64)
    return int(s[0]), int(s[1])


@dataclass
class Layout:
    rows: int
    cols: int
    row_perm: np.ndarray
    col_perm: np.ndarray
    row_cuts: np.ndarray
    col_cuts: np.ndarray
    block_size: int
    seed: int


def make_layout(a: sp.csr_matrix, procs: int, block_size=64, seed=0,
                permutation="block_random", partitioning="nnz",
                grid=None) -> Layout:
    """partition.py:216-254."""
    m, n = a.shape
    if grid is None:
        r, c = grid_shape(m, n, procs)
    else:
        r, c = max(min(grid[0], m), 1), max(min(grid[1], n), 1)
    rs, cs = axis_seeds(seed)
    if permutation == "none":
        rp, cp, b = np.arange(m), np.arange(n), block_size
    else:
        b = 1 if permutation == "full_random" else block_size
        rp, cp = shuffle_blocks(m, b, rs), shuffle_blocks(n, b, cs)
    if partitioning == "uniform":
        rc, cc = even_cuts(m, r), even_cuts(n, c)
    else:
        row_cnt = np.diff(a.indptr)
        col_cnt = np.bincount(a.indices, minlength=n)
        rc, cc = greedy_cuts(row_cnt[rp], r), greedy_cuts(col_cnt[cp], c)
    return Layout(r, c, np.asarray(rp, np.int64), np.asarray(cp, np.int64),
                  rc, cc, b, seed)


def permute_csr(a: sp.csr_matrix, lay: Layout) -> sp.csr_matrix:
    """partition.py:262-293 (row gather + column relabel + from_coo sort)."""
    m, n = a.shape
    inv_c = np.empty(n, dtype=np.int64)
    inv_c[lay.col_perm] = np.arange(n)
    lens = np.diff(a.indptr)[lay.row_perm]
    src = np.repeat(a.indptr[:-1][lay.row_perm] - (np.cumsum(lens) - lens), lens) \
        + np.arange(int(lens.sum()), dtype=np.int64)
    rows = np.repeat(np.arange(m, dtype=np.int64), lens)
    return csr_from_triplets(m, n, rows, inv_c[a.indices[src]], a.data[src])


def take_block(a: sp.csr_matrix, r0, r1, c0, c1) -> sp.csr_matrix:
    """sparse_kernels.py:48-58."""
    s = a[r0:r1, c0:c1].tocsr()
    s.sort_indices()
    return s


def unpermute(lay: Layout, xp: np.ndarray, yp: np.ndarray):
    """partition.py:322-337."""
    x = np.empty_like(xp)
    y = np.empty_like(yp)
    x[lay.col_perm] = xp
    y[lay.row_perm] = yp
    return x, y


def layout_summary(a: sp.csr_matrix, lay: Layout) -> dict:
    """partition.py:340-378."""
    R, C = lay.rows, lay.cols
    if a.nnz:
        inv_r = np.empty_like(lay.row_perm)
        inv_r[lay.row_perm] = np.arange(len(lay.row_perm))
        inv_c = np.empty_like(lay.col_perm)
        inv_c[lay.col_perm] = np.arange(len(lay.col_perm))
        er = np.repeat(np.arange(a.shape[0]), np.diff(a.indptr))
        br = np.searchsorted(lay.row_cuts, inv_r[er], side="right") - 1
        bc = np.searchsorted(lay.col_cuts, inv_c[a.indices], side="right") - 1
        per = np.bincount(br * C + bc, minlength=R * C)
    else:
        per = np.zeros(R * C, dtype=np.int64)
    devs = [{"i": i, "j": j,
             "rows": int(lay.row_cuts[i + 1] - lay.row_cuts[i]),
             "cols": int(lay.col_cuts[j + 1] - lay.col_cuts[j]),
             "nnz": int(per[i * C + j])} for i in range(R) for j in range(C)]
    f = per.astype(np.float64)
    mean = float(f.mean()) if len(f) else 0.0
    return {"grid": {"rows": R, "cols": C},
            "permutation": {"block_size": lay.block_size, "seed": lay.seed},
            "total_nnz": int(per.sum()),
            "nnz_max": int(f.max()) if len(f) else 0,
            "nnz_max_over_mean": float(f.max() / mean) if mean > 0 else 0.0,
            "devices": devs}


# ---------------------------------------------------------------------------
# per-block arithmetic (pdhg_engine.py:171-216)
# ---------------------------------------------------------------------------

def primal_map(x, c, aty, tau, lo, hi):
    return np.clip(x - tau * (c - aty), lo, hi)


def dual_map(y, z, sigma, clo, chi):
    v = y / sigma - z
    return sigma * (v - np.clip(v, -chi, -clo))


def anchor_mix(t, cur, anchor, k, gamma):
    wm = (1.0 + gamma) * (k + 1.0) / (k + 2.0)
    wa = 1.0 / (k + 2.0)
    return (wm * t - gamma * cur) + wa * anchor


def penalty(v, lo, hi) -> float:
    pos = np.maximum(v, 0.0)
    neg = np.maximum(-v, 0.0)
    fu, fl = np.isfinite(hi), np.isfinite(lo)
    if np.any(pos[~fu] > 0.0) or np.any(neg[~fl] > 0.0):
        return float("inf")
    return float(np.dot(hi[fu], pos[fu]) - np.dot(lo[fl], neg[fl]))


def range_gap(ax, clo, chi):
    return np.maximum(ax - chi, 0.0) - np.maximum(clo - ax, 0.0)


def gap_rel(p: float, d: float) -> float:
    if not math.isfinite(d) or not math.isfinite(p):
        return float("inf")
    return abs(p - d) / (1.0 + max(abs(p), abs(d)))


def pid_step(st: dict, dx: float, dy: float, omega: float, kp, ki, kd, lo, hi):
    """pdhg_engine.py:285-307 (state dict holds integral/last)."""
    if dx <= 0.0 or dy <= 0.0:
        return omega
    so = math.sqrt(omega)
    e = math.log((so * dx) / (dy / so))
    st["integral"] += e
    lw = math.log(omega) - (kp * e + ki * st["integral"] + kd * (e - st["last"]))
    st["last"] = e
    return min(max(math.exp(lw), lo), hi)


def restart_fires(base, r, prev, k, total, bs, bn, ba) -> bool:
    """pdhg_engine.py:262-282."""
    if base is not None:
        if r <= bs * base:
            return True
        if prev is not None and r <= bn * base and r > prev:
            return True
    return k >= ba * total


def probe_vector(n: int, seed: int) -> np.ndarray:
    """solver_driver.py:161-165."""
    return np.random.default_rng(np.random.SeedSequence(entropy=(seed, 0x5eed))).standard_normal(n)


def problem_norms(c, clo, chi) -> tuple[float, float]:
    """solver_driver.py:149-158: (||c||, ||finite bounds||), original order."""
    sq = float(np.sum(clo[np.isfinite(clo)] ** 2) + np.sum(chi[np.isfinite(chi)] ** 2))
    return float(np.linalg.norm(c)), math.sqrt(sq)


# ---------------------------------------------------------------------------
# lockstep grid simulation
# ---------------------------------------------------------------------------

def _asc(vals):
    """Ascending-order reduction (comm.py:75-84)."""
    acc = vals[0]
    if isinstance(acc, np.ndarray):
        acc = acc.copy()
        for v in vals[1:]:
            acc += v
    else:
        for v in vals[1:]:
            acc = acc + v
    return acc


@dataclass
class OracleResult:
    status: str
    x: np.ndarray
    y: np.ndarray
    r_primal: float
    r_dual: float
    r_gap: float
    obj_primal: float
    obj_dual: float
    objective: float
    iterations: int
    restarts: int
    eta: float
    omega: float
    passes: list = field(default_factory=list)   # per KKT pass tuples
    trace: dict = field(default_factory=dict)    # total -> (x_perm, y_perm)
    layout: dict = field(default_factory=dict)


DEFAULTS = dict(
    tolerance=1e-4, max_iterations=200_000, time_limit_seconds=None,
    kkt_interval=64, block_size=64, seed=0, n_procs=1, grid=None,
    permutation="block_random", partitioning="nnz", gamma=0.0, halpern=True,
    restarts=True, beta_sufficient=0.2, beta_necessary=0.8,
    beta_artificial=0.36, pid_kp=0.6, pid_ki=0.1, pid_kd=0.1,
    omega_min=1e-6, omega_max=1e6, omega_initial=None, eta=None,
    power_iterations=30,
)


class _Grid:
    """Blocks of the permuted problem on an R x C grid (partition.py:296-319)."""

    def __init__(self, problem, lay: Layout):
        a = as_csr(problem.matrix)
        self.lay = lay
        pa = permute_csr(a, lay)
        rp, cp = lay.row_perm, lay.col_perm
        self.R, self.C = lay.rows, lay.cols
        self.rr = [(int(lay.row_cuts[i]), int(lay.row_cuts[i + 1])) for i in range(self.R)]
        self.cr = [(int(lay.col_cuts[j]), int(lay.col_cuts[j + 1])) for j in range(self.C)]
        self.A = {}
        self.AT = {}
        for i, (r0, r1) in enumerate(self.rr):
            for j, (c0, c1) in enumerate(self.cr):
                blk = take_block(pa, r0, r1, c0, c1)
                self.A[i, j] = blk
                self.AT[i, j] = csr_transpose(blk)
        cvec = np.asarray(problem.objective, np.float64)[cp]
        lv = np.asarray(problem.var_lower, np.float64)[cp]
        uv = np.asarray(problem.var_upper, np.float64)[cp]
        lc = np.asarray(problem.con_lower, np.float64)[rp]
        uc = np.asarray(problem.con_upper, np.float64)[rp]
        self.c = [cvec[a0:a1].copy() for a0, a1 in self.cr]
        self.lv = [lv[a0:a1].copy() for a0, a1 in self.cr]
        self.uv = [uv[a0:a1].copy() for a0, a1 in self.cr]
        self.lc = [lc[a0:a1].copy() for a0, a1 in self.rr]
        self.uc = [uc[a0:a1].copy() for a0, a1 in self.rr]

    pool = None   # optional ThreadPoolExecutor: one host thread per block, like the
    #               reference's "threads" executor (comm.py:197-222); scipy releases
    #               the GIL so block products overlap. Results are unchanged.

    def _map(self, f, keys):
        if self.pool is None:
            return {k: f(k) for k in keys}
        return dict(zip(keys, self.pool.map(f, keys)))

    # axis-reduced products --------------------------------------------------
    def col_products(self, xs):
        """z_i = AllReduce_C(A_ij x_j), plus the partials."""
        keys = [(i, j) for i in range(self.R) for j in range(self.C)]
        part = self._map(lambda k: seq_spmv(self.A[k], xs[k[1]]), keys)
        red = [_asc([part[i, j] for j in range(self.C)]) for i in range(self.R)]
        return red, part

    def row_products(self, ys):
        """s_j = AllReduce_R(A_ij^T y_i)."""
        keys = [(i, j) for i in range(self.R) for j in range(self.C)]
        part = self._map(lambda k: seq_spmv(self.AT[k], ys[k[0]]), keys)
        return [_asc([part[i, j] for i in range(self.R)]) for j in range(self.C)]

    def g_sum(self, f):
        """AllReduce_G over ranks i*C+j in ascending order of f(i, j)."""
        return _asc([f(i, j) for i in range(self.R) for j in range(self.C)])


def _power(g: _Grid, iters: int, probe: np.ndarray) -> float:
    """sparse_kernels.py:61-93 on every block in lockstep (1x1 == :96-119)."""
    R, C = float(g.R), float(g.C)
    v = [np.asarray(probe[a0:a1], dtype=np.float64) for a0, a1 in g.cr]
    est = 0.0
    for _ in range(iters):
        u, _ = g.col_products(v)
        u_sq = g.g_sum(lambda i, j: float(np.dot(u[i], u[i])) / C)
        v_sq = g.g_sum(lambda i, j: float(np.dot(v[j], v[j])) / R)
        if u_sq == 0.0 or v_sq == 0.0:
            return 0.0
        est = math.sqrt(u_sq / v_sq)
        s = g.row_products(u)
        s_sq = g.g_sum(lambda i, j: float(np.dot(s[j], s[j])) / R)
        if s_sq == 0.0:
            return est
        v = [sj / math.sqrt(s_sq) for sj in s]
    return est


def _kkt(g: _Grid, xs, ys, tau, cnorm, bnorm, const):
    """pdhg_engine.py:310-346 in lockstep. Returns report tuple + reuse."""
    ax, part_ax = g.col_products(xs)
    rv = [range_gap(ax[i], g.lc[i], g.uc[i]) for i in range(g.R)]
    rp_sq = _asc([float(np.dot(rv[i], rv[i])) for i in range(g.R)])
    r_p = math.sqrt(rp_sq) / (1.0 + bnorm)

    aty = g.row_products(ys)
    shifted = [xs[j] - tau * (g.c[j] - aty[j]) for j in range(g.C)]
    xprobe = [np.clip(shifted[j], g.lv[j], g.uv[j]) for j in range(g.C)]
    rd = [(xprobe[j] - xs[j]) / tau for j in range(g.C)]
    rd_sq = _asc([float(np.dot(rd[j], rd[j])) for j in range(g.C)])
    r_d = math.sqrt(rd_sq) / (1.0 + cnorm)

    rc = [(xprobe[j] - shifted[j]) / tau for j in range(g.C)]
    obj_p = _asc([float(np.dot(g.c[j], xs[j])) for j in range(g.C)])
    pen = _asc([penalty(-ys[i], g.lc[i], g.uc[i]) for i in range(g.R)])
    cdot = _asc([float(np.dot(rc[j], xs[j])) for j in range(g.C)])
    obj_d = -pen + cdot
    rep = (r_p, r_d, gap_rel(obj_p, obj_d), obj_p + const, obj_d + const)
    return rep, part_ax, xprobe


def _broken(rep) -> bool:
    """pdhg_engine.py:356-361."""
    return (not math.isfinite(rep[0])) or (not math.isfinite(rep[1])) or math.isnan(rep[3])


def oracle_solve(problem, trace_at=(), **overrides) -> OracleResult:
    """Lockstep restatement of solve()/reference_solve(). Options are the
    SolverConfig fields (solver_driver.py:55-82)."""
    cfg = dict(DEFAULTS)
    unknown = set(overrides) - set(cfg)
    if unknown:
        raise TypeError(f"unknown options {sorted(unknown)}")
    cfg.update(overrides)
    a = as_csr(problem.matrix)
    lay = make_layout(a, cfg["n_procs"], cfg["block_size"], cfg["seed"],
                      cfg["permutation"], cfg["partitioning"], cfg["grid"])
    g = _Grid(problem, lay)
    c_orig = np.asarray(problem.objective, np.float64)
    cnorm, bnorm = problem_norms(c_orig, np.asarray(problem.con_lower, np.float64),
                                 np.asarray(problem.con_upper, np.float64))
    const = float(getattr(problem, "objective_constant", 0.0))
    probe = probe_vector(a.shape[1], cfg["seed"])
    est = _power(g, cfg["power_iterations"], probe)
    eta = cfg["eta"] if cfg["eta"] is not None else (0.998 / est if est > 0.0 else 1.0)
    if cfg["omega_initial"] is not None:
        omega = cfg["omega_initial"]
    elif cnorm > 0.0 and bnorm > 0.0:
        omega = cnorm / bnorm
    else:
        omega = 1.0
    R, C = g.R, g.C

    xs = [np.clip(np.zeros(c1 - c0), g.lv[j], g.uv[j]) for j, (c0, c1) in enumerate(g.cr)]
    ys = [np.zeros(r1 - r0) for r0, r1 in g.rr]
    x0 = [v.copy() for v in xs]
    y0 = [v.copy() for v in ys]
    k = 0
    epochs = 0
    total = 0
    base_fp = None
    prev_fp = None
    pid = {"integral": 0.0, "last": 0.0}
    status = None
    rep = None
    rep_at = -1
    passes = []
    trace = {}
    want = set(trace_at)
    gamma = cfg["gamma"]

    while True:
        if total >= cfg["max_iterations"]:
            status = ITER_LIMIT
            break
        tau, sigma = eta / omega, eta * omega
        aty = g.row_products(ys)
        xh = [primal_map(xs[j], g.c[j], aty[j], tau, g.lv[j], g.uv[j]) for j in range(C)]
        xb = [2.0 * xh[j] - xs[j] for j in range(C)]
        z, _ = g.col_products(xb)
        yh = [dual_map(ys[i], z[i], sigma, g.lc[i], g.uc[i]) for i in range(R)]
        if cfg["halpern"]:
            xs = [anchor_mix(xh[j], xs[j], x0[j], k, gamma) for j in range(C)]
            ys = [anchor_mix(yh[i], ys[i], y0[i], k, gamma) for i in range(R)]
        else:
            xs, ys = xh, yh
        k += 1
        total += 1
        if total in want:
            trace[total] = (np.concatenate(xs), np.concatenate(ys))
        if total % cfg["kkt_interval"] != 0:
            continue

        rep, part_ax, xprobe = _kkt(g, xs, ys, tau, cnorm, bnorm, const)
        rep_at = total
        passes.append((total,) + rep + (omega, eta, epochs))
        if _broken(rep):
            status = NUM_FAIL
            break
        if max(rep[0], rep[1], rep[2]) <= cfg["tolerance"]:
            status = OPTIMAL
            break

        if cfg["restarts"]:
            xbp = [2.0 * xprobe[j] - xs[j] for j in range(C)]
            zp, part_p = g.col_products(xbp)
            yp = [dual_map(ys[i], zp[i], sigma, g.lc[i], g.uc[i]) for i in range(R)]
            dx = [xs[j] - xprobe[j] for j in range(C)]
            dy = [ys[i] - yp[i] for i in range(R)]
            dx_sq = g.g_sum(lambda i, j: float(np.dot(dx[j], dx[j])) / float(R))
            dy_sq = g.g_sum(lambda i, j: float(np.dot(dy[i], dy[i])) / float(C))
            cross = g.g_sum(lambda i, j: float(np.dot(0.5 * (part_ax[i, j] - part_p[i, j]), dy[i])))
            val = (omega / eta) * dx_sq + dy_sq / (eta * omega) + 2.0 * cross
            fp = math.sqrt(max(val, 0.0))
            if base_fp is None:
                base_fp = fp
            if restart_fires(base_fp, fp, prev_fp, k, total, cfg["beta_sufficient"],
                             cfg["beta_necessary"], cfg["beta_artificial"]):
                ddx = g.g_sum(lambda i, j: float(np.dot(xs[j] - x0[j], xs[j] - x0[j])) / R)
                ddy = g.g_sum(lambda i, j: float(np.dot(ys[i] - y0[i], ys[i] - y0[i])) / C)
                omega = pid_step(pid, math.sqrt(ddx), math.sqrt(ddy), omega,
                                 cfg["pid_kp"], cfg["pid_ki"], cfg["pid_kd"],
                                 cfg["omega_min"], cfg["omega_max"])
                x0 = [v.copy() for v in xs]
                y0 = [v.copy() for v in ys]
                k = 0
                epochs += 1
                base_fp = fp
                prev_fp = None
            else:
                prev_fp = fp

    if rep_at != total:
        rep, _, _ = _kkt(g, xs, ys, eta / omega, cnorm, bnorm, const)
        if status != NUM_FAIL and _broken(rep):
            status = NUM_FAIL

    x, y = unpermute(lay, np.concatenate(xs) if xs else np.zeros(0),
                     np.concatenate(ys) if ys else np.zeros(0))
    obj = -rep[3] if getattr(problem, "maximize", False) else rep[3]
    return OracleResult(status=status, x=x, y=y, r_primal=rep[0], r_dual=rep[1],
                        r_gap=rep[2], obj_primal=rep[3], obj_dual=rep[4],
                        objective=obj, iterations=total, restarts=epochs,
                        eta=eta, omega=omega, passes=passes, trace=trace,
                        layout=layout_summary(a, lay))


def power_estimate(problem, seed=0, iters=30, **layout_opts) -> float:
    """Step-size estimate of the grid (solver_driver.py:211-227)."""
    a = as_csr(problem.matrix)
    lay = make_layout(a, layout_opts.get("n_procs", 1), layout_opts.get("block_size", 64),
                      seed, layout_opts.get("permutation", "block_random"),
                      layout_opts.get("partitioning", "nnz"), layout_opts.get("grid"))
    return _power(_Grid(problem, lay), iters, probe_vector(a.shape[1], seed))


def iteration_rate(problem, iters: int, grid=(1, 1), threads: int = 1, eta: float = 0.01,
                   seed: int = 0) -> dict:
    """Throughput of the reference's main-loop iteration (pdhg_engine.py:394-403,
    solver_driver.py:376-386) on the host: builds the grid blocks untimed, then
    times `iters` iterations (2 products + projections + Halpern per block).
    With threads > 1 the block products run on a thread pool, as the
    reference's threads executor does."""
    import time
    from concurrent.futures import ThreadPoolExecutor

    a = as_csr(problem.matrix)
    lay = make_layout(a, grid[0] * grid[1], 64, seed, "block_random", "nnz", tuple(grid))
    t0 = time.perf_counter()
    g = _Grid(problem, lay)
    setup = time.perf_counter() - t0
    if threads > 1:
        g.pool = ThreadPoolExecutor(max_workers=threads)
    R, C = g.R, g.C
    omega = 1.0
    xs = [np.clip(np.zeros(c1 - c0), g.lv[j], g.uv[j]) for j, (c0, c1) in enumerate(g.cr)]
    ys = [np.zeros(r1 - r0) for r0, r1 in g.rr]
    x0 = [v.copy() for v in xs]
    y0 = [v.copy() for v in ys]
    tau, sigma = eta / omega, eta * omega
    # with a pool the per-block epilogues run on it too (numpy releases the
    # GIL), as each device's whole iteration does in the reference's threads
    # executor (comm.py:185-221)
    pmap = (lambda f, n: list(g.pool.map(f, range(n)))) if g.pool is not None else (
        lambda f, n: [f(q) for q in range(n)])
    t0 = time.perf_counter()
    for k in range(iters):
        aty = g.row_products(ys)

        def primal(j):
            xh = primal_map(xs[j], g.c[j], aty[j], tau, g.lv[j], g.uv[j])
            return xh, 2.0 * xh - xs[j]
        pj = pmap(primal, C)
        xh = [h for h, _ in pj]
        xb = [b for _, b in pj]
        z, _ = g.col_products(xb)
        yh = pmap(lambda i: dual_map(ys[i], z[i], sigma, g.lc[i], g.uc[i]), R)
        xs = pmap(lambda j: anchor_mix(xh[j], xs[j], x0[j], k, 0.0), C)
        ys = pmap(lambda i: anchor_mix(yh[i], ys[i], y0[i], k, 0.0), R)
    dt = time.perf_counter() - t0
    if g.pool is not None:
        g.pool.shutdown()
    return {"iterations": iters, "seconds": dt, "iters_per_s": iters / dt if dt > 0 else float("inf"),
            "setup_seconds": setup, "grid": [R, C], "threads": threads}
