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
DEFAULT_VARIANT = 9


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
    info[pos] = (slen[pos] << 8) | (order[pos] & (window - 1))
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

    variant 9 (default; 10 = early epilogue loads): SELL-32 with one-warp
    windows; variants 6-8: SELL-32 with 256-row windows — only the SELL
    arrays and the heavy-row CSR live in HBM, built either on the host
    (build_sell, from a HostCsr) or on the device (DeviceSetup.sell, passed
    as a dict). Variants 0-5: tiled CSR (tile directory + int32 CSR), kept
    for A/B measurement."""

    PAD = 4   # the TMA staging copies read whole 16-byte granules

    def __init__(self, host: HostCsr, device, exact_row_max: int = DEFAULT_EXACT_ROW_MAX,
                 tile_cap: int = native.DEFAULT_TILE_CAP, variant: int = DEFAULT_VARIANT):
        if isinstance(host, dict):
            shape = host["shape"]
            self.num_rows, self.num_cols, self.nnz = shape
            lens = np.zeros(0, dtype=np.int64)
            self.heavy_rows = int(len(host["heavy_rows"]))
        else:
            if host.nnz >= 2 ** 31 - 64:
                raise ValueError("block nnz must be < 2^31 (int32 offsets)")
            self.num_rows, self.num_cols, self.nnz = host.num_rows, host.num_cols, host.nnz
            lens = np.diff(host.ptr)
            self.heavy_rows = int(np.count_nonzero(lens > exact_row_max))
        self.exact_row_max, self.tile_cap, self.variant = exact_row_max, tile_cap, variant
        # the host copy is kept only for CPU-resident blocks (the CPU test double)
        self.host = host if torch.device(device).type == "cpu" else None
        self.dev = {}
        up = lambda k, a: self.dev.__setitem__(k, torch.from_numpy(np.ascontiguousarray(a)).to(device))  # noqa: E731
        ptr = lambda k: self.dev[k].data_ptr() if k in self.dev and self.dev[k].numel() else None  # noqa: E731
        csr_args = [None, None, None, None, 0, None, 0, None, 0]
        sell_args = [None] * 4 + [0] + [None] * 4 + [0]
        self.num_tiles = 0
        if variant >= 6:
            if isinstance(host, dict):      # SELL arrays already built on the device (DeviceSetup.sell)
                sd = host
                for k in ("vals", "cols", "slice_off", "lane_info", "heavy_rows", "heavy_ptr", "heavy_cols",
                          "heavy_vals"):
                    self.dev["sell_" + k] = sd[k]
            else:
                sd = build_sell(host, exact_row_max, window=32 if variant >= 9 else SELL_WINDOW)
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
        if self.variant >= 9:
            return (self.num_windows + 1) // 2 + self.heavy_rows
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


@dataclass
class DeviceCsrArrays:
    """A block (or its transpose) as int32 CSR in HBM — the output of the
    device setup, input of the SELL build."""

    num_rows: int
    num_cols: int
    nnz: int
    ptr: torch.Tensor
    col: torch.Tensor
    val: torch.Tensor


class DeviceSetup:
    """One-off device preprocessing through the C ABI (csrc/gridlp_setup.cu):
    the original CSR is uploaded once; every local block is then extracted
    (permuted, column-banded, rows sorted by column), transposed and laid
    out as SELL-32 on the device. Replaces the host permute/slice/transpose
    (partition.py:262-319, sparse_kernels.py:27-58)."""

    def __init__(self, problem, layout, device):
        self.lib = native.load()
        self.device = device
        self.layout = layout
        A = problem.matrix
        m, n = int(A.num_rows), int(A.num_cols)
        if n >= 2 ** 31 - 1 or m >= 2 ** 31 - 1:
            raise ValueError("device setup needs < 2^31 rows and columns per matrix")
        nnz = int(len(A.values))

        def t(a, dt):
            return torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(device)

        self.src_ptr = t(A.row_offsets, np.int64)
        self.src_col = t(A.col_indices, np.int32) if nnz else torch.zeros(1, dtype=torch.int32, device=device)
        self.src_val = t(A.values, np.float64) if nnz else torch.zeros(1, dtype=torch.float64, device=device)
        self.inv_col = t(layout.perm.inverse_cols(), np.int32) if n else torch.zeros(1, dtype=torch.int32,
                                                                                      device=device)
        self.row_perm = t(layout.perm.row_perm, np.int64) if m else torch.zeros(1, dtype=torch.int64,
                                                                                 device=device)
        items = max(nnz, m + n) + 64
        segs = (m + n) + (m + n) // 32 + 64
        wsb = int(self.lib._lib.gridlp_setup_workspace_bytes(items, segs))
        self.ws = torch.empty(wsb, dtype=torch.uint8, device=device)
        self.ws_bytes = wsb
        self.h2d_bytes = sum(x.numel() * x.element_size()
                             for x in (self.src_ptr, self.src_col, self.src_val, self.inv_col, self.row_perm))

    def _stream(self):
        return torch.cuda.current_stream(self.device).cuda_stream

    def block(self, i: int, j: int) -> DeviceCsrArrays:
        lay = self.layout
        r0, r1 = lay.row_range(i)
        c0, c1 = lay.col_range(j)
        nrows = r1 - r0
        band = self.row_perm[r0:r1]
        ptr = torch.empty(nrows + 1, dtype=torch.int32, device=self.device)
        self.lib.call("gridlp_block_count", self.src_ptr.data_ptr(), self.src_col.data_ptr(),
                      band.data_ptr() if nrows else None, nrows, self.inv_col.data_ptr(), c0, c1,
                      ptr.data_ptr(), self.ws.data_ptr(), self.ws_bytes, self._stream())
        nnz = int(ptr[-1].item())
        col = torch.empty(nnz + 8, dtype=torch.int32, device=self.device)
        val = torch.empty(nnz + 8, dtype=torch.float64, device=self.device)
        self.lib.call("gridlp_block_fill", self.src_ptr.data_ptr(), self.src_col.data_ptr(),
                      self.src_val.data_ptr(), band.data_ptr() if nrows else None, nrows,
                      self.inv_col.data_ptr(), c0, c1, ptr.data_ptr(), nnz, col.data_ptr(), val.data_ptr(),
                      self.ws.data_ptr(), self.ws_bytes, self._stream())
        return DeviceCsrArrays(nrows, c1 - c0, nnz, ptr, col, val)

    def transpose(self, a: DeviceCsrArrays) -> DeviceCsrArrays:
        ptr = torch.empty(a.num_cols + 1, dtype=torch.int32, device=self.device)
        col = torch.empty(a.nnz + 8, dtype=torch.int32, device=self.device)
        val = torch.empty(a.nnz + 8, dtype=torch.float64, device=self.device)
        self.lib.call("gridlp_csr_transpose", a.ptr.data_ptr(), a.col.data_ptr(), a.val.data_ptr(), a.num_rows,
                      a.num_cols, a.nnz, ptr.data_ptr(), col.data_ptr(), val.data_ptr(), self.ws.data_ptr(),
                      self.ws_bytes, self._stream())
        return DeviceCsrArrays(a.num_cols, a.num_rows, a.nnz, ptr, col, val)

    def sell(self, a: DeviceCsrArrays, exact_row_max: int) -> dict:
        """SELL-32 warp-window arrays (variants 9/10) built on the device."""
        dev, m = self.device, a.num_rows
        ns = (m + 31) // 32
        i32 = dict(dtype=torch.int32, device=dev)
        lane_info = torch.empty(max(ns * 32, 1), **i32)
        slice_off = torch.empty(ns + 1, **i32)
        rank_of = torch.empty(max(m, 1), **i32)
        heavy_rows = torch.empty(max(m, 1), **i32)
        heavy_ptr = torch.empty(m + 1, **i32)
        sizes = torch.zeros(3, dtype=torch.int64, device=dev)
        self.lib.call("gridlp_sell_plan", a.ptr.data_ptr(), m, exact_row_max, lane_info.data_ptr(),
                      slice_off.data_ptr(), rank_of.data_ptr(), heavy_rows.data_ptr(), heavy_ptr.data_ptr(),
                      sizes.data_ptr(), self.ws.data_ptr(), self.ws_bytes, self._stream())
        total, nh, hnnz = (int(v) for v in sizes.cpu().tolist())
        sell_col = torch.empty(total + 8, **i32)
        sell_val = torch.empty(total + 8, dtype=torch.float64, device=dev)
        hcol = torch.empty(hnnz + 8, **i32)
        hval = torch.empty(hnnz + 8, dtype=torch.float64, device=dev)
        self.lib.call("gridlp_sell_fill", a.ptr.data_ptr(), a.col.data_ptr(), a.val.data_ptr(), m, exact_row_max,
                      slice_off.data_ptr(), rank_of.data_ptr(), heavy_rows.data_ptr(), heavy_ptr.data_ptr(), nh,
                      sell_col.data_ptr(), sell_val.data_ptr(), total, hcol.data_ptr(), hval.data_ptr(),
                      self._stream())
        return dict(vals=sell_val, cols=sell_col, slice_off=slice_off, lane_info=lane_info,
                    num_windows=ns, heavy_rows=heavy_rows[:nh].clone() if nh else heavy_rows[:0],
                    heavy_ptr=heavy_ptr[: nh + 1].clone(), heavy_cols=hcol, heavy_vals=hval)

    def release(self):
        for name in ("src_ptr", "src_col", "src_val", "inv_col", "row_perm", "ws"):
            setattr(self, name, None)
