"""Per-device blocks: permutation, 2D slicing, stored transpose, tiling, and
upload into HBM.

Reference: permute_problem / distribute (partition.py:262-319), slice_block
and transpose (sparse_kernels.py:27-58). The reference builds CSR with int64
indices (16 B/nnz); a device block here stores int32 row pointers and column
indices with FP64 values (12 B/nnz per orientation) plus a tile directory
(include/gridlp_b200.h, gridlp_csr_t).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import native

DEFAULT_EXACT_ROW_MAX = 512
DEFAULT_VARIANT = 6


@dataclass
class HostCsr:
    num_rows: int
    num_cols: int
    ptr: np.ndarray   # int64 [rows+1]
    col: np.ndarray   # int64 [nnz]
    val: np.ndarray   # f64 [nnz]

    @property
    def nnz(self) -> int:
        return int(len(self.val))


def _csr_arrays(matrix):
    return (np.asarray(matrix.row_offsets, dtype=np.int64),
            np.asarray(matrix.col_indices, dtype=np.int64),
            np.asarray(matrix.values, dtype=np.float64))


def permute_matrix(matrix, layout) -> HostCsr:
    """Rows gathered in permuted order, columns relabelled, each row's
    entries ordered by new column (== the reference's from_coo lexsort)."""
    off, col, val = _csr_arrays(matrix)
    m, n = int(matrix.num_rows), int(matrix.num_cols)
    rp = layout.perm.row_perm
    inv_c = layout.perm.inverse_cols()
    lens = np.diff(off)[rp]
    total = int(lens.sum())
    new_ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    if total == 0:
        return HostCsr(m, n, new_ptr, np.zeros(0, np.int64), np.zeros(0))
    src = np.repeat(off[:-1][rp] - new_ptr[:-1], lens) + np.arange(total, dtype=np.int64)
    ncol = inv_c[col[src]]
    rows = np.repeat(np.arange(m, dtype=np.int64), lens)
    order = np.argsort(rows * max(n, 1) + ncol, kind="stable")
    return HostCsr(m, n, new_ptr, ncol[order], val[src][order])


def slice_blocks(pa: HostCsr, layout) -> dict:
    """{(i, j): HostCsr} of A_ij with local indices (sparse_kernels.py:48-58)."""
    R, C = layout.topology.rows, layout.topology.cols
    out = {}
    band_of_col = np.searchsorted(layout.col_cuts, pa.col, side="right") - 1
    for i in range(R):
        r0, r1 = layout.row_range(i)
        e0, e1 = int(pa.ptr[r0]), int(pa.ptr[r1])
        rows_local = np.repeat(np.arange(r1 - r0, dtype=np.int64), np.diff(pa.ptr[r0:r1 + 1]))
        bands = band_of_col[e0:e1]
        for j in range(C):
            c0, c1 = layout.col_range(j)
            sel = np.flatnonzero(bands == j) + e0 if C > 1 else np.arange(e0, e1)
            lr = rows_local[sel - e0]
            ptr = np.concatenate([[0], np.cumsum(np.bincount(lr, minlength=r1 - r0))]).astype(np.int64)
            out[(i, j)] = HostCsr(r1 - r0, c1 - c0, ptr, pa.col[sel] - c0, pa.val[sel])
    return out


def transpose(a: HostCsr) -> HostCsr:
    """Explicit transpose with sorted columns (sparse_kernels.py:27-36)."""
    rows = np.repeat(np.arange(a.num_rows, dtype=np.int64), np.diff(a.ptr))
    order = np.argsort(a.col * max(a.num_rows, 1) + rows, kind="stable")
    ptr = np.concatenate([[0], np.cumsum(np.bincount(a.col, minlength=a.num_cols))]).astype(np.int64)
    return HostCsr(a.num_cols, a.num_rows, ptr, rows[order], a.val[order])


def build_tiles(ptr: np.ndarray, exact_row_max: int = DEFAULT_EXACT_ROW_MAX,
                cap: int = native.TILE_NNZ_CAP, max_rows: int = native.TILE_ROWS) -> np.ndarray:
    """Tile directory for the product kernel.

    Light tiles group the rows whose first nonzero falls in the same window
    of (cap - exact_row_max) nonzeros, so a light tile never exceeds `cap`
    nonzeros, and are split further to at most `max_rows` rows. Every row
    longer than exact_row_max is isolated in its own (heavy) tile.
    """
    ptr = np.asarray(ptr, dtype=np.int64)
    m = len(ptr) - 1
    if m <= 0:
        return np.zeros(1, dtype=np.int32)
    if not (0 <= exact_row_max <= cap // 2):
        raise ValueError("exact_row_max must be in [0, cap/2]")
    seg = cap - exact_row_max
    lens = np.diff(ptr)
    heavy = lens > exact_row_max
    win = ptr[:-1] // seg
    start = np.zeros(m, dtype=bool)
    start[0] = True
    start[1:] = win[1:] != win[:-1]
    start |= heavy
    start[1:] |= heavy[:-1]
    run = np.cumsum(start) - 1
    first = np.flatnonzero(start)
    pos = np.arange(m, dtype=np.int64) - first[run]
    start |= (pos % max_rows) == 0
    tiles = np.concatenate([np.flatnonzero(start), [m]]).astype(np.int64)
    if tiles[-1] >= 2 ** 31:
        raise ValueError("too many rows for int32 tiles")
    return tiles.astype(np.int32)


SELL_WINDOW = 256


def build_sell(host: HostCsr, exact_row_max: int, window: int = SELL_WINDOW):
    """SELL-32 layout of include/gridlp_b200.h (variant 6): per 256-row
    window the light rows sorted by length (descending, stable) into 32-lane
    slices stored column-major; heavy rows as a compact CSR."""
    ptr, m = host.ptr, host.num_rows
    lens = np.diff(ptr)
    heavy = lens > exact_row_max
    nw = -(-m // window) if m else 0
    eff = np.where(heavy, -1, lens)
    win = np.arange(m, dtype=np.int64) // window
    order = np.lexsort((-eff, win))             # window-major, longest first, heavy last
    info = np.full(nw * window, -1, dtype=np.int64)
    slen = eff[order]
    light = slen >= 0
    pos = np.flatnonzero(light)
    info[pos] = (slen[pos] << 8) | (order[pos] & 255)
    lane_len = np.zeros(nw * window, dtype=np.int64)
    lane_len[pos] = slen[pos]
    slice_len = lane_len.reshape(-1, 32).max(axis=1) if nw else np.zeros(0, np.int64)
    slice_off = np.concatenate([[0], np.cumsum(32 * slice_len)]).astype(np.int64)
    total = int(slice_off[-1])
    if total >= 2 ** 31 - 64:
        raise ValueError("SELL block too large for int32 offsets")
    vals = np.zeros(total + 8, dtype=np.float64)
    cols = np.zeros(total + 8, dtype=np.int32)
    rows_l = order[pos]
    cnt = lens[rows_l]
    base = slice_off[pos // 32] + (pos % 32)
    nl = int(cnt.sum())
    if nl:
        first = np.repeat(np.cumsum(cnt) - cnt, cnt)
        j = np.arange(nl, dtype=np.int64) - first
        dest = np.repeat(base, cnt) + 32 * j
        src = np.repeat(ptr[rows_l], cnt) + j
        vals[dest] = host.val[src]
        cols[dest] = host.col[src]
    hrows = np.flatnonzero(heavy).astype(np.int64)
    hlen = lens[hrows]
    hptr = np.concatenate([[0], np.cumsum(hlen)]).astype(np.int64)
    if len(hrows):
        hsrc = np.repeat(ptr[hrows] - hptr[:-1], hlen) + np.arange(int(hptr[-1]), dtype=np.int64)
        hcols = np.concatenate([host.col[hsrc].astype(np.int32), np.zeros(4, np.int32)])
        hvals = np.concatenate([host.val[hsrc], np.zeros(4)])
    else:
        hcols, hvals = np.zeros(4, np.int32), np.zeros(4)
    return dict(vals=vals, cols=cols, slice_off=slice_off.astype(np.int32),
                lane_info=info.astype(np.int32), num_windows=nw, heavy_rows=hrows.astype(np.int32),
                heavy_ptr=hptr.astype(np.int32), heavy_cols=hcols, heavy_vals=hvals)


class DeviceCsr:
    """One block resident in HBM; `.struct` is its gridlp_csr_t.

    variant >= 6 (default 6): SELL-32 windows (build_sell) — only the SELL
    arrays and the heavy-row CSR are uploaded. variants 0-5: tiled CSR
    (tile directory + int32 CSR), kept for A/B measurement."""

    PAD = 4   # the TMA staging copies read whole 16-byte granules

    def __init__(self, host: HostCsr, device, exact_row_max: int = DEFAULT_EXACT_ROW_MAX,
                 tile_cap: int = native.DEFAULT_TILE_CAP, variant: int = DEFAULT_VARIANT):
        if host.nnz >= 2 ** 31 - 64:
            raise ValueError("block nnz must be < 2^31 (int32 offsets)")
        self.num_rows, self.num_cols, self.nnz = host.num_rows, host.num_cols, host.nnz
        self.exact_row_max, self.tile_cap, self.variant = exact_row_max, tile_cap, variant
        # the host copy is kept only for CPU-resident blocks (the CPU test double)
        self.host = host if torch.device(device).type == "cpu" else None
        self.dev = {}
        up = lambda k, a: self.dev.__setitem__(k, torch.from_numpy(np.ascontiguousarray(a)).to(device))  # noqa: E731
        ptr = lambda k: self.dev[k].data_ptr() if k in self.dev and self.dev[k].numel() else None  # noqa: E731
        lens = np.diff(host.ptr)
        self.heavy_rows = int(np.count_nonzero(lens > exact_row_max))
        csr_args = [None, None, None, None, 0, None, 0, None, 0]
        sell_args = [None] * 4 + [0] + [None] * 4 + [0]
        self.num_tiles = 0
        if variant >= 6:
            sd = build_sell(host, exact_row_max)
            for k in ("vals", "cols", "slice_off", "lane_info", "heavy_rows", "heavy_ptr", "heavy_cols",
                      "heavy_vals"):
                up("sell_" + k, sd[k])
            sell_args = [ptr("sell_vals"), ptr("sell_cols"), ptr("sell_slice_off"), ptr("sell_lane_info"),
                         sd["num_windows"], ptr("sell_heavy_rows"), ptr("sell_heavy_ptr"),
                         ptr("sell_heavy_cols"), ptr("sell_heavy_vals"), len(sd["heavy_rows"])]
            self.num_windows = sd["num_windows"]
        else:
            tiles = build_tiles(host.ptr, exact_row_max, cap=tile_cap)
            self.num_tiles = max(len(tiles) - 1, 0)
            t_rows = np.diff(tiles.astype(np.int64))
            first = tiles[:-1].astype(np.int64)
            heavy = (t_rows == 1) & (lens[first] > exact_row_max) if self.num_tiles else np.zeros(0, bool)
            col = np.zeros(host.nnz + self.PAD, dtype=np.int32)
            col[: host.nnz] = host.col
            val = np.zeros(host.nnz + self.PAD, dtype=np.float64)
            val[: host.nnz] = host.val
            up("row_ptr", host.ptr.astype(np.int32))
            up("col_idx", col)
            up("values", val)
            up("tile_ptr", tiles)
            up("light_tiles", np.flatnonzero(~heavy).astype(np.int32))
            up("heavy_tiles", np.flatnonzero(heavy).astype(np.int32))
            csr_args = [ptr("row_ptr"), ptr("col_idx"), ptr("values"), ptr("tile_ptr"), self.num_tiles,
                        ptr("light_tiles"), int(np.count_nonzero(~heavy)), ptr("heavy_tiles"),
                        int(np.count_nonzero(heavy))]
        self.struct = native.Csr(self.num_rows, self.num_cols, self.nnz, *csr_args, *sell_args,
                                 exact_row_max, tile_cap, variant, 0)

    def tensors(self):
        return tuple(self.dev.values())

    def slots(self) -> int:
        if self.variant >= 6:
            return self.num_windows + self.heavy_rows
        return self.num_tiles

    def src(self, gather: torch.Tensor | None) -> native.Src:
        s = native.Src()
        s.A = ctypes.pointer(self.struct)
        s.gather = gather.data_ptr() if gather is not None and gather.numel() else None
        s.nparts = 0
        s.num_rows = self.num_rows
        return s

    def bytes_per_product(self) -> int:
        """Algorithmic bytes of one product: 12/nnz + row pointers + one read
        of the gathered vector + one FP64 result per row."""
        return 12 * self.nnz + 4 * (self.num_rows + 1) + 8 * self.num_cols + 8 * self.num_rows


def parts_src(parts, num_rows: int) -> native.Src:
    """Source summing partial vectors in ascending order (comm.py:75-84)."""
    if len(parts) > native.MAX_PARTS:
        raise ValueError(f"at most {native.MAX_PARTS} partial vectors per reduction")
    s = native.Src()
    s.A = None
    s.gather = None
    for q, p in enumerate(parts):
        s.parts[q] = p.data_ptr() if p.numel() else None
    s.nparts = len(parts)
    s.num_rows = num_rows
    return s
