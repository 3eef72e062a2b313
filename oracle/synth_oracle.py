"""TEST INFRASTRUCTURE — numpy restatement of the device generators
(paper_2601_07628_b200/csrc/gridlp_gen.cu, driven by synth.py).

These generators have no counterpart in the reference (generators.py:23
lists block_diagonal, staircase, uniform_random, box_lp_known_optimum), so
there is no reference output to pin against: "parity unpinned" with respect
to the reference; the contract is internal — the device instance must equal
this restatement bit for bit — and the feasibility construction follows the
reference's uniform_random wrapper (generators.py:120-142: box bounds,
rhs = A x_hat by sequential csr_matvec, a fraction of rows ranged by
U[0.1, 1) on each side).

Only tests/ may import this module. Everything here is written from the
formulas in include/gridlp_b200.h (device generators section), not from the
CUDA code, with numpy uint64 wrap-around arithmetic for the hash and plain
IEEE float64 operations in the same order for every derived number.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

M1 = np.uint64(0x9E3779B97F4A7C15)
M2 = np.uint64(0xBF58476D1CE4E5B9)
M3 = np.uint64(0x94D049BB133111EB)


def mix(z):
    with np.errstate(over="ignore"):
        z = z + M1
        z = (z ^ (z >> np.uint64(30))) * M2
        z = (z ^ (z >> np.uint64(27))) * M3
    return z ^ (z >> np.uint64(31))


def u01(seed, stream, a, b=0):
    with np.errstate(over="ignore"):
        s = mix(np.uint64(seed) * np.uint64(0x100000001B3) + np.uint64(stream))
    h = mix(mix(s ^ np.asarray(a, dtype=np.uint64)) ^ np.asarray(b, dtype=np.uint64))
    return (h >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def powerlaw(m, n, nnz_target, alpha=0.8, ineq=0.3, box=(0.0, 4.0), seed=0):
    """Returns dict(ptr, col, val, x_hat, c, var_lo, var_hi, con_lo, con_hi)."""
    w = (np.arange(m, dtype=np.float64) + 1.0) ** -alpha
    d = np.clip(np.floor(float(nnz_target) * (w / w.sum()) + u01(seed, 0, np.arange(m))).astype(np.int64), 1, n)
    rows = np.repeat(np.arange(m, dtype=np.int64), d)
    k = np.arange(int(d.sum()), dtype=np.int64) - np.repeat(np.cumsum(d) - d, d)
    u = u01(seed, 1, rows, k)
    kappa = (n + 1.0) ** 0.2 - 1.0
    a = 1.0 + u * kappa
    t = a * a * a * a * a
    c = np.clip(np.floor(t).astype(np.int64) - 1, 0, n - 1)
    key = np.unique(rows * n + c)                 # sorted, distinct (row, col)
    r, col = key // n, key % n
    val = 2.0 * u01(seed, 2, r, col) - 1.0
    ptr = np.concatenate([[0], np.cumsum(np.bincount(r, minlength=m))]).astype(np.int64)
    x_hat = 1.0 + (3.0 - 1.0) * u01(seed, 3, np.arange(n))
    cvec = -1.0 + (1.0 - -1.0) * u01(seed, 4, np.arange(n))
    b = sp.csr_matrix((val, col, ptr), shape=(m, n)).dot(x_hat)
    ranged = u01(seed, 5, np.arange(m)) < ineq
    wl = 0.1 + 0.9 * u01(seed, 6, np.arange(m))
    wh = 0.1 + 0.9 * u01(seed, 7, np.arange(m))
    lo = np.where(ranged, b - wl, b)
    hi = np.where(ranged, b + wh, b)
    return dict(ptr=ptr, col=col, val=val, x_hat=x_hat, c=cvec, var_lo=np.full(n, box[0]),
                var_hi=np.full(n, box[1]), con_lo=lo, con_hi=hi)


def mcf(V, E, K, capacity_factor=1.25, seed=0):
    e = np.arange(E)
    tail = np.floor(u01(seed, 10, e) * V).astype(np.int64)
    head = (tail + 1 + np.floor(u01(seed, 11, e) * (V - 1)).astype(np.int64)) % V
    m, n = K * V + E, K * E
    rows, cols, vals = [], [], []
    for k in range(K):
        # conservation rows (k, v): +1 on out-arcs, -1 on in-arcs
        rows += [k * V + tail, k * V + head]
        cols += [k * E + e, k * E + e]
        vals += [np.ones(E), -np.ones(E)]
        rows.append(K * V + e)                       # coupling row of arc e
        cols.append(k * E + e)
        vals.append(np.ones(E))
    A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(m, n)).tocsr()
    A.sort_indices()
    x_hat = 0.5 + (1.5 - 0.5) * u01(seed, 12, np.arange(n))
    cvec = 1.0 + (10.0 - 1.0) * u01(seed, 13, np.arange(n))
    b = A.dot(x_hat)
    lo, hi = b.copy(), b.copy()
    lo[K * V:] = -np.inf
    hi[K * V:] = b[K * V:] * capacity_factor
    return dict(ptr=A.indptr.astype(np.int64), col=A.indices.astype(np.int64), val=A.data, x_hat=x_hat, c=cvec,
                var_lo=np.zeros(n), var_hi=np.full(n, 4.0), con_lo=lo, con_hi=hi)


def planted(m, n, d, box=(0.0, 4.0), seed=0):
    """Planted-optimum LP (cfg5 generator): dict as powerlaw() plus y_star."""
    rows = np.repeat(np.arange(m, dtype=np.int64), d)
    k = np.tile(np.arange(d, dtype=np.int64), m)
    c = np.floor(u01(seed, 1, rows, k) * float(n)).astype(np.int64)
    c = np.minimum(c, n - 1)
    key = np.unique(rows * n + c)
    r, col = key // n, key % n
    val = 2.0 * u01(seed, 2, r, col) - 1.0
    ptr = np.concatenate([[0], np.cumsum(np.bincount(r, minlength=m))]).astype(np.int64)
    A = sp.csr_matrix((val, col, ptr), shape=(m, n))
    j = np.arange(n)
    st = u01(seed, 20, j)
    w = 0.1 + 0.9 * u01(seed, 21, j)
    lo, hi = box
    x = np.where(st < 0.3, lo, np.where(st < 0.4, hi, lo + (hi - lo) * (0.1 + 0.8 * u01(seed, 22, j))))
    rc = np.where(st < 0.3, w, np.where(st < 0.4, -w, 0.0))
    b = A.dot(x)
    i = np.arange(m)
    sti = u01(seed, 23, i)
    yv = 0.5 + u01(seed, 24, i)
    wl = 0.1 + 0.9 * u01(seed, 25, i)
    wh = 0.1 + 0.9 * u01(seed, 26, i)
    y = np.where(sti < 0.35, yv, np.where(sti < 0.7, -yv, 0.0))
    clo = np.where(sti < 0.35, b, b - wl)
    chi = np.where(sti < 0.35, b + wl, np.where(sti < 0.7, b, b + wh))
    t = A.T.tocsr()
    t.sort_indices()
    cvec = t.dot(y) + rc
    return dict(ptr=ptr, col=col, val=val, x_hat=x, c=cvec, var_lo=np.full(n, lo), var_hi=np.full(n, hi),
                con_lo=clo, con_hi=chi, y_star=y)
