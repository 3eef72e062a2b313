"""Grid layout: topology choice, block-wise random permutation and
nonzero-balanced cuts (host integer work, bit-identical to the reference).

Reference: /root/reference/pkg/src/gridlp/partition.py:24-378 —
select_grid :131-150, block_random_permutation :153-173, uniform_cuts
:176-179, nnz_balanced_cuts :182-206, build_layout :216-254, _axis_seeds
:257-259, unpermute_solution :322-337, layout_summary :340-378.

Device (i, j) of an R x C grid owns A_ij = rows [row_cuts[i], row_cuts[i+1])
x cols [col_cuts[j], col_cuts[j+1]) of the permuted matrix; primal vectors
are replicated down grid column j, dual vectors across grid row i.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

PERMUTATIONS = ("none", "full_random", "block_random")
PARTITIONINGS = ("uniform", "nnz")


@dataclass(frozen=True)
class GridTopology:
    rows: int
    cols: int

    def __post_init__(self):
        if self.rows < 1 or self.cols < 1:
            raise ValueError("grid dimensions must be positive")

    @property
    def num_devices(self) -> int:
        return self.rows * self.cols

    def coords(self):
        return [(i, j) for i in range(self.rows) for j in range(self.cols)]


def invert_permutation(perm: np.ndarray) -> np.ndarray:
    inv = np.empty_like(perm)
    inv[perm] = np.arange(len(perm), dtype=perm.dtype)
    return inv


@dataclass(frozen=True)
class Permutation:
    """perm[k] = original index placed at permuted position k."""

    row_perm: np.ndarray
    col_perm: np.ndarray
    block_size: int
    seed: int

    def inverse_rows(self) -> np.ndarray:
        return invert_permutation(self.row_perm)

    def inverse_cols(self) -> np.ndarray:
        return invert_permutation(self.col_perm)


@dataclass(frozen=True)
class PartitionLayout:
    topology: GridTopology
    perm: Permutation
    row_cuts: np.ndarray
    col_cuts: np.ndarray

    def __post_init__(self):
        for name, parts in (("row_cuts", self.topology.rows), ("col_cuts", self.topology.cols)):
            arr = np.ascontiguousarray(getattr(self, name), dtype=np.int64)
            if arr.shape != (parts + 1,) or arr[0] != 0 or np.any(np.diff(arr) < 0):
                raise ValueError(f"{name} must be non-decreasing with {parts + 1} entries from 0")
            object.__setattr__(self, name, arr)

    @property
    def num_rows(self) -> int:
        return int(self.row_cuts[-1])

    @property
    def num_cols(self) -> int:
        return int(self.col_cuts[-1])

    def row_range(self, i) -> tuple[int, int]:
        return int(self.row_cuts[i]), int(self.row_cuts[i + 1])

    def col_range(self, j) -> tuple[int, int]:
        return int(self.col_cuts[j]), int(self.col_cuts[j + 1])


def select_grid(m: int, n: int, n_procs: int) -> GridTopology:
    """Most devices used, then grid aspect closest to m/n in log space, then
    the taller grid (partition.py:131-150)."""
    if n_procs < 1:
        raise ValueError("n_procs must be >= 1")
    aim = math.log(max(m, 1) / max(n, 1))
    col_cap = max(min(n_procs, n), 1)
    candidates = []
    for r in range(1, max(min(n_procs, m), 1) + 1):
        c = min(n_procs // r, col_cap)
        if c >= 1:
            candidates.append(((-r * c, abs(math.log(r / c) - aim), -r), r, c))
    _, r, c = min(candidates, key=lambda t: t[0])
    return GridTopology(r, c)


def block_random_permutation(length: int, block_size: int, seed: int) -> np.ndarray:
    """Fisher-Yates over contiguous blocks of `block_size` indices, order kept
    inside a block (partition.py:153-173). The bounded draws for positions
    nb-1..1 are taken in one vectorised call, which numpy's Generator
    produces identically to one `integers(0, i+1)` call per position."""
    if block_size < 1:
        raise ValueError("block_size must be >= 1")
    if length == 0:
        return np.empty(0, dtype=np.int64)
    nb = -(-length // block_size)
    draws = np.random.default_rng(seed).integers(0, np.arange(nb, 1, -1)) if nb > 1 else []
    order = list(range(nb))
    for i, k in zip(range(nb - 1, 0, -1), draws.tolist() if nb > 1 else []):
        order[i], order[k] = order[k], order[i]
    order = np.asarray(order, dtype=np.int64)
    first = order * block_size
    width = np.minimum(first + block_size, length) - first
    offset = np.repeat(first - (np.cumsum(width) - width), width)
    return offset + np.arange(length, dtype=np.int64)


def _check_parts(length: int, parts: int):
    if parts < 1:
        raise ValueError("parts must be >= 1")
    if parts > length and not (length == 0 and parts == 1):
        raise ValueError(f"cannot split {length} indices into {parts} non-empty parts")


def uniform_cuts(length: int, parts: int) -> np.ndarray:
    """Cut t at ceil(t * length / parts) (partition.py:176-179)."""
    _check_parts(length, parts)
    return np.array([-(-t * length // parts) for t in range(parts + 1)], dtype=np.int64)


def nnz_balanced_cuts(counts, parts: int) -> np.ndarray:
    """Greedy nonzero-balanced boundaries (partition.py:182-206).

    The reference sweeps index by index; the boundary it stops at is the
    first prefix length whose running sum reaches total*p/parts, clamped so
    every earlier part keeps >= 1 index and every later part can too. That
    closed form is evaluated here with a prefix sum + searchsorted.
    """
    counts = np.asarray(counts)
    if np.any(counts < 0):
        raise ValueError("counts must be non-negative")
    length = len(counts)
    _check_parts(length, parts)
    if length == 0:
        return np.zeros(parts + 1, dtype=np.int64)
    prefix = np.concatenate([[0], np.cumsum(counts.astype(np.int64))])
    total = int(prefix[-1])
    cuts = [0]
    for p in range(1, parts):
        goal = total * p / parts          # Python float, as in the reference
        first = int(np.searchsorted(prefix, goal, side="left"))
        cut = max(cuts[-1] + 1, first)
        cut = min(cut, length - (parts - p))
        cuts.append(cut)
    cuts.append(length)
    return np.array(cuts, dtype=np.int64)


def axis_seeds(seed: int) -> tuple[int, int]:
    """Row/column permutation seeds (partition.py:257-259)."""
    st = np.random.SeedSequence(seed).generate_state(2, dtype=np.uint64)
    return int(st[0]), int(st[1])


def _row_counts(matrix) -> np.ndarray:
    return np.diff(np.asarray(matrix.row_offsets, dtype=np.int64))


def _col_counts(matrix) -> np.ndarray:
    return np.bincount(np.asarray(matrix.col_indices, dtype=np.int64),
                       minlength=int(matrix.num_cols)).astype(np.int64)


def build_layout(problem, n_procs: int, block_size: int = 64, seed: int = 0,
                 permutation: str = "block_random", partitioning: str = "nnz",
                 grid: GridTopology | None = None) -> PartitionLayout:
    """partition.py:216-254."""
    if permutation not in PERMUTATIONS:
        raise ValueError(f"unknown permutation strategy {permutation!r}")
    if partitioning not in PARTITIONINGS:
        raise ValueError(f"unknown partitioning strategy {partitioning!r}")
    A = problem.matrix
    m, n = int(A.num_rows), int(A.num_cols)
    if grid is None:
        grid = select_grid(m, n, n_procs)
    else:
        grid = GridTopology(max(min(grid.rows, m), 1), max(min(grid.cols, n), 1))
    rseed, cseed = axis_seeds(seed)
    if permutation == "none":
        rp, cp, b = np.arange(m, dtype=np.int64), np.arange(n, dtype=np.int64), block_size
    else:
        b = 1 if permutation == "full_random" else block_size
        rp = block_random_permutation(m, b, rseed)
        cp = block_random_permutation(n, b, cseed)
    perm = Permutation(rp, cp, b, seed)
    if partitioning == "uniform":
        rc, cc = uniform_cuts(m, grid.rows), uniform_cuts(n, grid.cols)
    else:
        # one part needs no counts: the cut is [0, length] (skips an nnz-long bincount)
        rc = nnz_balanced_cuts(_row_counts(A)[rp], grid.rows) if grid.rows > 1 else np.array([0, m], np.int64)
        cc = nnz_balanced_cuts(_col_counts(A)[cp], grid.cols) if grid.cols > 1 else np.array([0, n], np.int64)
    return PartitionLayout(grid, perm, rc, cc)


def unpermute_solution(layout: PartitionLayout, x_blocks, y_blocks):
    """Concatenate grid-column x blocks / grid-row y blocks and return them in
    original index order (partition.py:322-337)."""
    xp = np.concatenate([np.asarray(b, dtype=np.float64) for b in x_blocks]) if x_blocks else np.empty(0)
    yp = np.concatenate([np.asarray(b, dtype=np.float64) for b in y_blocks]) if y_blocks else np.empty(0)
    if xp.shape != (layout.num_cols,):
        raise ValueError("primal blocks do not cover the column cuts")
    if yp.shape != (layout.num_rows,):
        raise ValueError("dual blocks do not cover the row cuts")
    x = np.empty_like(xp)
    y = np.empty_like(yp)
    x[layout.perm.col_perm] = xp
    y[layout.perm.row_perm] = yp
    return x, y


def layout_summary(problem, layout: PartitionLayout, per_device_nnz=None) -> dict:
    """JSON-ready per-device sizes and nonzero counts (partition.py:340-378).
    `per_device_nnz` (row-major) may be supplied when the blocks are already
    built; otherwise it is counted from the original matrix."""
    R, C = layout.topology.rows, layout.topology.cols
    if per_device_nnz is None:
        A = problem.matrix
        if int(np.asarray(A.row_offsets)[-1]) if int(A.num_rows) else 0:
            inv_r = layout.perm.inverse_rows()
            inv_c = layout.perm.inverse_cols()
            band_r = np.searchsorted(layout.row_cuts, inv_r, side="right") - 1
            band_c = np.searchsorted(layout.col_cuts, inv_c, side="right") - 1
            rows_of = np.repeat(band_r, _row_counts(A))
            per = np.bincount(rows_of * C + band_c[np.asarray(A.col_indices)], minlength=R * C)
        else:
            per = np.zeros(R * C, dtype=np.int64)
    else:
        per = np.asarray(per_device_nnz, dtype=np.int64)
    devices = []
    for i in range(R):
        r0, r1 = layout.row_range(i)
        for j in range(C):
            c0, c1 = layout.col_range(j)
            devices.append({"i": i, "j": j, "rows": r1 - r0, "cols": c1 - c0,
                            "nnz": int(per[i * C + j])})
    f = per.astype(np.float64)
    mean = float(f.mean()) if len(f) else 0.0
    return {
        "grid": {"rows": R, "cols": C},
        "permutation": {"block_size": layout.perm.block_size, "seed": layout.perm.seed},
        "total_nnz": int(per.sum()),
        "nnz_max": int(f.max()) if len(f) else 0,
        "nnz_max_over_mean": float(f.max() / mean) if mean > 0 else 0.0,
        "devices": devices,
    }
