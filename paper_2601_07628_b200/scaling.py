"""Diagonal preconditioning on the device: Ruiz equilibration followed by
Pock-Chambolle scaling (alpha = 1), the preconditioner of cuPDLP — north-star
item 4 / SURVEY §8f rank 3. The reference solves the unscaled problem
(SPEC.md:64), so this is opt-in through SolverConfig.scaling; the default
("none") keeps bit parity with the reference.

The scaled LP is  min (Dc c)ᵀ x'  s.t.  Dr lc <= (Dr A Dc) x' <= Dr uc,
lv / Dc <= x' <= uv / Dc, and the solution maps back as x = Dc x',
y = Dr y'. Ruiz iteration k divides every row and column by the square
root of its largest |a|; Pock-Chambolle then divides row i by
sqrt(sum_j |a_ij|) and column j by sqrt(sum_i |a_ij|). Every step is a
kernel of csrc/gridlp_scale.cu; the reductions are deterministic (order-free
maxima, sequential sums along rows of A and of its transpose), so a scaled
solve is run-to-run reproducible. oracle/scaling_oracle.py restates the same
arithmetic in numpy.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import native
from .problem import LpProblem, SparseMatrix

MODES = ("none", "ruiz", "pock_chambolle", "ruiz+pock_chambolle")


class _ScaledMatrix:
    """The scaled CSR as the solver sees it: the sparsity pattern on the host
    (the layout needs only counts) and the scaled values on the device (the
    device setup consumes them there). `values` downloads on first access
    (nothing on the solve path reads it)."""

    def __init__(self, A, dev_val, nnz):
        self.num_rows, self.num_cols = int(A.num_rows), int(A.num_cols)
        self.row_offsets, self.col_indices = A.row_offsets, A.col_indices
        self._dev_val, self._nnz, self._host = dev_val, nnz, None

    @property
    def values(self):
        if self._host is None:
            self._host = self._dev_val[:self._nnz].cpu().numpy()
        return self._host

    @property
    def nnz(self):
        return self._nnz

    @property
    def shape(self):
        return (self.num_rows, self.num_cols)


@dataclass
class ScaledProblem:
    problem: LpProblem          # the scaled LP (solve() input; matrix values stay on the device)
    row_scale: np.ndarray       # Dr
    col_scale: np.ndarray       # Dc
    seconds: float = 0.0
    device_csr: tuple | None = None     # (ptr int64, col int32, val f64) of the scaled A in HBM
    row_scale_device: object = None
    col_scale_device: object = None

    def unscale(self, x: np.ndarray, y: np.ndarray):
        return x * self.col_scale, y * self.row_scale


def scale_problem(problem, mode: str = "ruiz+pock_chambolle", ruiz_iterations: int = 10,
                  device=None) -> ScaledProblem:
    if mode not in MODES or mode == "none":
        raise ValueError(f"scaling mode must be one of {MODES[1:]}")
    import time

    t0 = time.perf_counter()
    lib = native.load()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream(dev).cuda_stream
    A = problem.matrix
    m, n, nnz = int(A.num_rows), int(A.num_cols), int(len(A.values))
    if n >= 2 ** 31 or nnz >= 2 ** 31:
        raise ValueError("device scaling needs < 2^31 columns and nonzeros")
    f64 = dict(dtype=torch.float64, device=dev)
    ptr = torch.from_numpy(np.ascontiguousarray(A.row_offsets, np.int64)).to(dev)
    col = torch.from_numpy(np.ascontiguousarray(A.col_indices, np.int32)).to(dev) if nnz else torch.zeros(
        1, dtype=torch.int32, device=dev)
    val = torch.from_numpy(np.ascontiguousarray(A.values, np.float64)).to(dev) if nnz else torch.zeros(1, **f64)
    dr, dc = torch.ones(m, **f64), torch.ones(n, **f64)
    sr, sc = torch.empty(m, **f64), torch.empty(n, **f64)
    rstat, cstat = torch.empty(max(m, 1), **f64), torch.empty(max(n, 1), **f64)
    p = lambda t: t.data_ptr()  # noqa: E731

    def apply():
        lib.call("gridlp_update_scale", p(rstat), m, p(dr), p(sr), stream)
        lib.call("gridlp_update_scale", p(cstat), n, p(dc), p(sc), stream)
        lib.call("gridlp_scale_matrix", p(ptr), p(col), p(val), m, p(sr), p(sc), stream)

    if mode in ("ruiz", "ruiz+pock_chambolle"):
        for _ in range(ruiz_iterations):
            lib.call("gridlp_row_absmax", p(ptr), p(val), m, p(rstat), stream)
            lib.call("gridlp_col_absmax", p(col), p(val), nnz, n, p(cstat), stream)
            apply()
    if mode in ("pock_chambolle", "ruiz+pock_chambolle"):
        lib.call("gridlp_row_abssum", p(ptr), p(val), m, 1, p(rstat), stream)
        # column sums run along the rows of the transpose (rows ascending inside a column)
        wsb = int(lib._lib.gridlp_setup_workspace_bytes(nnz + 64, max(m, n) + 64))
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        p32 = ptr.to(torch.int32)
        tptr = torch.empty(n + 1, dtype=torch.int32, device=dev)
        tcol = torch.empty(nnz + 8, dtype=torch.int32, device=dev)
        tval = torch.empty(nnz + 8, **f64)
        lib.call("gridlp_csr_transpose", p(p32), p(col), p(val), m, n, nnz, p(tptr), p(tcol), p(tval), p(ws), wsb,
                 stream)
        lib.call("gridlp_row_abssum", p(tptr.to(torch.int64)), p(tval), n, 1, p(cstat), stream)
        del ws, p32, tcol, tval
        apply()
    c = torch.from_numpy(np.ascontiguousarray(problem.objective, np.float64)).to(dev)
    lv = torch.from_numpy(np.ascontiguousarray(problem.var_lower, np.float64)).to(dev)
    uv = torch.from_numpy(np.ascontiguousarray(problem.var_upper, np.float64)).to(dev)
    lc = torch.from_numpy(np.ascontiguousarray(problem.con_lower, np.float64)).to(dev)
    uc = torch.from_numpy(np.ascontiguousarray(problem.con_upper, np.float64)).to(dev)
    for v, d, div, k in ((c, dc, 0, n), (lv, dc, 1, n), (uv, dc, 1, n), (lc, dr, 0, m), (uc, dr, 0, m)):
        if k:
            lib.call("gridlp_scale_vector", p(v), p(d), k, div, stream)
    h = lambda t: t.cpu().numpy()  # noqa: E731
    scaled = LpProblem(SparseMatrix(m, n, A.row_offsets, A.col_indices, np.zeros(0), check=False),
                       h(c), h(lv), h(uv), h(lc), h(uc),
                       objective_constant=float(getattr(problem, "objective_constant", 0.0)),
                       maximize=bool(getattr(problem, "maximize", False)),
                       name=str(getattr(problem, "name", "")))
    # the scaled values never leave the device: the engine's device setup
    # takes the scaled CSR as its preloaded input
    scaled.matrix = _ScaledMatrix(A, val, nnz)
    torch.cuda.synchronize(dev)
    return ScaledProblem(scaled, h(dr), h(dc), time.perf_counter() - t0, device_csr=(ptr, col, val),
                         row_scale_device=dr, col_scale_device=dc)
