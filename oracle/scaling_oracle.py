"""TEST INFRASTRUCTURE — numpy restatement of the on-device diagonal
preconditioner (paper_2601_07628_b200/scaling.py, csrc/gridlp_scale.cu).

The reference has no scaling: parity is unpinned with respect
to the reference; the contract is that the device factors and the scaled
matrix equal this restatement bit for bit (maxima are exact, 1/sqrt is
correctly rounded in both, sums are sequential along rows of A / rows of
Aᵀ, and every product is taken in the same order). Only tests/ import it.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def _seq_row_sums(a: sp.csr_matrix) -> np.ndarray:
    out = np.zeros(a.shape[0])
    for r in range(a.shape[0]):
        seg = np.abs(a.data[a.indptr[r]:a.indptr[r + 1]])
        if len(seg):
            out[r] = np.add.accumulate(seg)[-1]          # left to right from the first entry
    return out


def _inv_sqrt(s):
    f = np.ones_like(s)
    pos = s > 0
    f[pos] = 1.0 / np.sqrt(s[pos])
    return f


def scale(ptr, col, val, m, n, mode="ruiz+pock_chambolle", ruiz_iterations=10):
    """Returns (scaled values in CSR entry order, Dr, Dc)."""
    a = sp.csr_matrix((np.asarray(val, np.float64).copy(), np.asarray(col), np.asarray(ptr)), shape=(m, n))
    rows = np.repeat(np.arange(m), np.diff(a.indptr))
    dr, dc = np.ones(m), np.ones(n)

    def apply(rs, cs):
        nonlocal dr, dc
        fr, fc = _inv_sqrt(rs), _inv_sqrt(cs)
        dr, dc = dr * fr, dc * fc
        a.data[:] = (fr[rows] * a.data) * fc[a.indices]

    if mode in ("ruiz", "ruiz+pock_chambolle"):
        for _ in range(ruiz_iterations):
            absd = np.abs(a.data)
            rs = np.zeros(m)
            np.maximum.at(rs, rows, absd)
            cs = np.zeros(n)
            np.maximum.at(cs, a.indices, absd)
            apply(rs, cs)
    if mode in ("pock_chambolle", "ruiz+pock_chambolle"):
        rs = _seq_row_sums(a)
        t = a.T.tocsr()
        t.sort_indices()
        cs = _seq_row_sums(t)
        apply(rs, cs)
    return a.data.copy(), dr, dc
