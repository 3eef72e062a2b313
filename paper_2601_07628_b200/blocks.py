"""Per-device blocks: permutation, 2D slicing, stored transpose, SELL-32
layout, and upload into HBM.

Reference: permute_problem / distribute (partition.py:262-319), slice_block
and transpose (sparse_kernels.py:27-58). The reference builds CSR with int64
indices (16 B/nnz); a device block here is SELL-32 with int32 column indices
and FP64 values (12 B/nnz per orientation) plus a compact CSR of its long
rows (include/gridlp_b200.h, gridlp_csr_t). Values that are all exactly
floats, or all +-1, are stored in the narrower lossless codecs
(GRIDLP_VALS_F32: 8 B/nnz, GRIDLP_VALS_UNIT: 4 B/nnz) — the kernels rebuild
the exact FP64 value, so products are unchanged bit for bit.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import native

DEFAULT_LIGHT_ROW_MAX = 128     # SELL-32 lanes (one lane per row); sweep in profiles/r1/row_classes.md
LIGHT_ROW_CANDIDATES = (128, 256, 512, 1024, 2048)   # the engine's per-block choices (profiles/r1/layout_autotune.md)
DEFAULT_EXACT_ROW_MAX = 4096    # one warp per row, still sequential sums; longer rows are chunked
WIDE_CTA_MAX_MEAN_ROW = 6.0     # mean light-row length at or below which SELL lanes use 4-warp CTAs


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


def permute_csr(a: HostCsr, row_order=None, col_label=None) -> HostCsr:
    """Host twin of gridlp_csr_permute: out row r = row row_order[r], column
    c relabelled col_label[c], entry order kept (row sums unchanged)."""
    lens = np.diff(a.ptr)
    order = np.arange(a.num_rows) if row_order is None else np.asarray(row_order, np.int64)
    nl = lens[order]
    ptr = np.concatenate([[0], np.cumsum(nl)]).astype(np.int64)
    src = np.repeat(a.ptr[:-1][order] - ptr[:-1], nl) + np.arange(int(ptr[-1]), dtype=np.int64)
    col = a.col[src] if col_label is None else np.asarray(col_label, np.int64)[a.col[src]]
    return HostCsr(a.num_rows, a.num_cols, ptr, col, a.val[src])


LENGTH_BUCKETS_PER_OCTAVE = 8


def length_order(lens: np.ndarray) -> np.ndarray:
    """Internal order of a band: rows grouped by length class, longest class
    first, layout order inside a class (stable). Classes are
    floor(8 log2(len + 1)) — about 9 % wide — so a SELL-32 slice holds rows
    within ~9 % of each other's length, the longest slices start first
    (LPT-like, no tail), and rows of one class keep their layout order, which
    preserves the gather locality of structured matrices (consecutive rows of
    one commodity in a flow LP). numpy's stable sort on the uint16 class key
    is a radix sort."""
    lens = np.asarray(lens, np.int64)
    cls = np.floor(LENGTH_BUCKETS_PER_OCTAVE * np.log2(lens.astype(np.float64) + 1.0)).astype(np.int64)
    return np.argsort((65535 - np.minimum(cls, 65535)).astype(np.uint16), kind="stable")


def length_order_device(lens: torch.Tensor) -> torch.Tensor:
    """length_order on the device (int64 indices): the same classes
    floor(8 log2(len + 1)), longest class first, stable inside a class."""
    cls = torch.floor(LENGTH_BUCKETS_PER_OCTAVE * torch.log2(lens.to(torch.float64) + 1.0)).to(torch.int64)
    return torch.sort(-cls, stable=True).indices


def inverse_order_device(order: torch.Tensor) -> torch.Tensor:
    inv = torch.empty_like(order)
    inv[order] = torch.arange(order.numel(), dtype=order.dtype, device=order.device)
    return inv


def inverse_order(order: np.ndarray) -> np.ndarray:
    inv = np.empty_like(order)
    inv[order] = np.arange(len(order), dtype=order.dtype)
    return inv


def build_sell(host: HostCsr, light_row_max: int):
    """SELL-32 layout of include/gridlp_b200.h on the host (the device build,
    DeviceSetup.sell, must produce the same arrays): per 32-row slice, lane l
    holds row 32 s + l (empty when the row is long), entries stored
    column-major; rows longer than light_row_max as a compact CSR."""
    ptr, m = host.ptr, host.num_rows
    lens = np.diff(ptr)
    heavy = lens > light_row_max
    ns = -(-m // 32) if m else 0
    eff = np.where(heavy, -1, lens)
    sl = np.arange(m, dtype=np.int64) // 32
    order = np.arange(m, dtype=np.int64)       # lane = row & 31
    info = np.full(ns * 32, -1, dtype=np.int64)
    slen = eff[order]
    light = slen >= 0
    pos = np.flatnonzero(light)
    info[pos] = (slen[pos] << 8) | (order[pos] & 31)
    lane_len = np.zeros(ns * 32, dtype=np.int64)
    lane_len[pos] = slen[pos]
    slice_len = lane_len.reshape(-1, 32).max(axis=1) if ns else np.zeros(0, np.int64)
    slice_off = np.concatenate([[0], np.cumsum(32 * slice_len)]).astype(np.int64)
    total = int(slice_off[-1])
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
    return dict(vals=vals, cols=cols, slice_off=slice_off.astype(np.int64),
                lane_info=info.astype(np.int32), num_slices=ns, long_rows=hrows.astype(np.int32),
                long_ptr=hptr.astype(np.int32), long_cols=hcols, long_vals=hvals)


def long_row_plan(long_ptr: torch.Tensor, exact_row_max: int):
    """Split the compact CSR's long rows: rows of length <= exact_row_max are
    summed exactly by one warp each (exact_long lists them in row order, so
    neighbouring warps gather neighbouring data); longer rows are
    cut into GRIDLP_HEAVY_CHUNK-entry chunks. Returns int32 tensors
    (exact_long, chunk_first [nl+1], chunk_row [num_chunks]) on long_ptr's
    device."""
    hp = long_ptr.to(torch.int64)
    nl = hp.numel() - 1
    lens = hp[1:] - hp[:-1]
    heavy = lens > exact_row_max
    nch = torch.where(heavy, (lens + native.HEAVY_CHUNK - 1) // native.HEAVY_CHUNK, torch.zeros_like(lens))
    first = torch.zeros(nl + 1, dtype=torch.int64, device=hp.device)
    if nl:
        first[1:] = torch.cumsum(nch, 0)
    rows = torch.repeat_interleave(torch.arange(nl, device=hp.device), nch) if nl else first[:0]
    if int(first[-1]) >= 2 ** 31:
        raise ValueError("too many heavy-row chunks for int32")
    exact = torch.nonzero(~heavy).flatten() if nl else first[:0]
    return exact.to(torch.int32), first.to(torch.int32), rows.to(torch.int32)


CODEC_NAMES = {native.VALS_F64: "f64", native.VALS_F32: "f32", native.VALS_UNIT: "unit"}
_CODEC_OF = {v: k for k, v in CODEC_NAMES.items()}
_CODEC_CHUNK = 1 << 26          # values examined per pass (bounds the temporaries on 2B-nnz blocks)
_SIGN32 = -(2 ** 31)


def value_codec_of(vals) -> int:
    """Narrowest lossless storage of a block's values (numpy or torch, the
    real entries only): GRIDLP_VALS_UNIT when every value is +1.0 or -1.0,
    GRIDLP_VALS_F32 when every value survives float32 exactly (NaN and
    subnormals do not), else GRIDLP_VALS_F64."""
    if isinstance(vals, np.ndarray):
        vals = torch.from_numpy(np.ascontiguousarray(vals, dtype=np.float64))
    n = int(vals.numel())
    unit = f32 = True
    for a in range(0, n, _CODEC_CHUNK):
        v = vals[a: a + _CODEC_CHUNK]
        if unit:
            unit = bool(((v == 1.0) | (v == -1.0)).all())
        if not unit:
            f32 = bool((v.float().double() == v).all())
            if not f32:
                break
    return native.VALS_UNIT if unit else native.VALS_F32 if f32 else native.VALS_F64


class DeviceCsr:
    """One block resident in HBM; `.struct` is its gridlp_csr_t.

    Built from a HostCsr (host SELL build, build_sell) or from the dict the
    device setup returns (DeviceSetup.sell). Only the SELL arrays, the heavy
    rows' chunked CSR and the chunk scratch live in HBM."""

    def __init__(self, host, device, exact_row_max: int = DEFAULT_EXACT_ROW_MAX,
                 light_row_max: int = DEFAULT_LIGHT_ROW_MAX, value_codec: str = "f64"):
        if not 0 <= light_row_max <= exact_row_max <= native.ROW_MAX_LIMIT:
            raise ValueError(f"need 0 <= light_row_max <= exact_row_max <= {native.ROW_MAX_LIMIT}")
        if isinstance(host, dict):      # SELL arrays already built on the device (DeviceSetup.sell)
            self.num_rows, self.num_cols, self.nnz = host["shape"]
            sd = host
            if sd.get("light_row_max", light_row_max) != light_row_max:
                raise ValueError("device SELL arrays were built for another light_row_max")
        else:
            if host.nnz >= 2 ** 31 - 64:
                raise ValueError("block nnz must be < 2^31 (int32 offsets)")
            self.num_rows, self.num_cols, self.nnz = host.num_rows, host.num_cols, host.nnz
            sd = build_sell(host, light_row_max)
        self.exact_row_max, self.light_row_max = exact_row_max, light_row_max
        # the host copy is kept only for CPU-resident blocks (the CPU test double)
        self.host = host if torch.device(device).type == "cpu" and not isinstance(host, dict) else None
        self.dev = {}
        for k in ("vals", "cols", "slice_off", "lane_info", "long_rows", "long_ptr", "long_cols", "long_vals"):
            a = sd[k]
            self.dev[k] = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a)).to(device)
        self.long_rows = int(self.dev["long_rows"].numel())
        self.dev["exact_long"], self.dev["chunk_first"], self.dev["chunk_row"] = long_row_plan(
            self.dev["long_ptr"], exact_row_max)
        self.num_exact_long = int(self.dev["exact_long"].numel())
        self.num_chunks = int(self.dev["chunk_row"].numel())
        self.heavy_rows = self.long_rows - self.num_exact_long
        self.dev["chunk_sums"] = torch.zeros(max(self.num_chunks, 1), dtype=torch.float64, device=device)
        self.dev["chunk_done"] = torch.zeros(max(self.long_rows, 1), dtype=torch.int32, device=device)
        self.num_slices = int(sd["num_slices"])
        self.val_codec = native.VALS_F64
        if value_codec != "f64" and self.nnz and torch.device(device).type == "cuda":
            real = sd["src_vals"] if isinstance(host, dict) else host.val
            self._apply_codec(value_codec, real)
        ptr = lambda k: self.dev[k].data_ptr() if self.dev[k].numel() else None  # noqa: E731
        self.struct = native.Csr(self.num_rows, self.num_cols, self.nnz,
                                 ptr("vals"), ptr("cols"), ptr("slice_off"), ptr("lane_info"), self.num_slices,
                                 ptr("long_rows"), ptr("long_ptr"), ptr("long_cols"), ptr("long_vals"),
                                 self.long_rows, ptr("exact_long"), self.num_exact_long,
                                 ptr("chunk_first"), ptr("chunk_row"), self.num_chunks, ptr("chunk_sums"),
                                 ptr("chunk_done"), light_row_max, exact_row_max)
        self.struct.val_codec = self.val_codec
        # launch hint: blocks of very short light rows (network / MCF columns)
        # run the main-loop SELL lanes in 4-warp CTAs (fewer CTA launches;
        # cfg4's A^T 2652 -> 2441 us, cfg2 / cfg3 rows of 10-20 stay at 2)
        if self.nnz and self.num_rows and torch.device(device).type == "cuda":
            hnnz = int(self.dev["long_ptr"][-1].item()) if self.long_rows else 0
            light_rows = self.num_rows - self.long_rows
            if light_rows > 0 and (self.nnz - hnnz) / light_rows <= WIDE_CTA_MAX_MEAN_ROW:
                self.struct.launch_flags |= native.CSR_WIDE_CTAS

    def _apply_codec(self, want: str, real):
        """Re-store the values in codec `want` ("auto": the narrowest lossless
        one; "f32" / "unit": forced, ValueError if not lossless). UNIT folds
        the sign into bit 31 of the column indices (padding entries are never
        read) and drops the value arrays; F32 narrows them."""
        if want not in ("auto", "f32", "unit"):
            raise ValueError(f"value_codec must be 'auto', 'f64', 'f32' or 'unit', not {want!r}")
        best = value_codec_of(real)
        if want != "auto":
            need = _CODEC_OF[want]
            if need > best:
                raise ValueError(f"value_codec={want!r} is not lossless for this block's values")
            best = need
        if best == native.VALS_UNIT:
            for vk, ck in (("vals", "cols"), ("long_vals", "long_cols")):
                v, c = self.dev[vk], self.dev[ck]
                for a in range(0, int(v.numel()), _CODEC_CHUNK):
                    neg = (v[a: a + _CODEC_CHUNK] < 0).to(torch.int32).mul_(_SIGN32)
                    c[a: a + _CODEC_CHUNK].bitwise_or_(neg)
                self.dev[vk] = v[:0]
        elif best == native.VALS_F32:
            for vk in ("vals", "long_vals"):
                self.dev[vk] = self.dev[vk].float()
        self.val_codec = best

    @property
    def codec(self) -> str:
        return CODEC_NAMES[self.val_codec]

    def tensors(self):
        return tuple(self.dev.values())

    def slots(self) -> int:
        """CTAs of one product (= reduction slots): heavy chunks + long-row
        warp pairs + slice pairs."""
        if not self.num_rows:
            return 0
        return self.num_chunks + (self.num_exact_long + 1) // 2 + (self.num_slices + 1) // 2

    def launches(self) -> int:
        """Kernels one product launches (heavy / long / SELL, when present)."""
        return int(self.num_chunks > 0) + int(self.num_exact_long > 0) + 1

    def src(self, gather: torch.Tensor | None) -> native.Src:
        s = native.Src()
        s.A = ctypes.pointer(self.struct)
        s.gather = gather.data_ptr() if gather is not None and gather.numel() else None
        s.nparts = 0
        s.num_rows = self.num_rows
        return s

    def bytes_per_product(self) -> int:
        """Algorithmic bytes of one product: 12/nnz (8 / 4 with the F32 / UNIT
        value codecs) + row pointers + one read of the gathered vector + one
        FP64 result per row."""
        per = 4 + (8, 4, 0)[self.val_codec]
        return per * self.nnz + 4 * (self.num_rows + 1) + 8 * self.num_cols + 8 * self.num_rows


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


class BandedCsr:
    """A block stored as K column bands (include/gridlp_b200.h, gridlp_csr_t
    .carry): band k holds each row's entries with columns in
    [cuts[k], cuts[k+1]) in their original order, rows over the full block.
    A product runs band by band — bands 0..K-2 store running row sums into
    `acc`, band k > 0 continues every row's add chain from acc — so each
    band's slice of the gather vector stays L2-resident and the sums are the
    unbanded ones bit for bit. Chunked rows (> exact_row_max) sit wholly in
    the last band. ops.CudaOps.src issues the leading bands."""

    def __init__(self, bands, cuts, device):
        if len(bands) < 2:
            raise ValueError("a banded block needs >= 2 bands")
        self.bands = list(bands)
        self.cuts = list(cuts)
        b0 = self.bands[0]
        self.num_rows, self.num_cols = b0.num_rows, b0.num_cols
        self.nnz = sum(b.nnz for b in self.bands)
        self.light_row_max = self.bands[-1].light_row_max
        self.acc = torch.zeros(max(self.num_rows, 1), dtype=torch.float64, device=device)
        for b in self.bands[1:]:
            b.struct.carry = self.acc.data_ptr()

    def tensors(self):
        return tuple(t for b in self.bands for t in b.tensors()) + (self.acc,)

    def slots(self) -> int:
        return max(b.slots() for b in self.bands)

    def launches(self) -> int:
        return sum(b.launches() for b in self.bands)

    def src(self, gather):
        return self.bands[-1].src(gather)


def split_column_bands(arr, cuts, exact_row_max: int, to_layout=None):
    """DeviceCsrArrays -> one DeviceCsrArrays per column band (torch ops on
    the device; entry order inside a row kept). Rows longer than
    exact_row_max go wholly to the last band. Bands are ranges of the
    LAYOUT column index, along which every row's entries ascend: with
    `to_layout` (internal column -> layout column, the engine's length-class
    order) the band of an entry is that of its layout column, so each band is
    still a contiguous piece of every row's add chain; its internal columns
    form one contiguous run per length class, a band's share of x̄."""
    dev = arr.col.device
    m, nnz = arr.num_rows, arr.nnz
    lens = (arr.ptr[1:] - arr.ptr[:-1]).long()
    row_of = torch.repeat_interleave(torch.arange(m, device=dev), lens)
    col = arr.col[:nnz]
    val = arr.val[:nnz]
    inner = torch.as_tensor(list(cuts[1:-1]), dtype=torch.int32, device=dev)
    key = col if to_layout is None else to_layout[col.long()].to(torch.int32)
    band = torch.bucketize(key, inner, right=True)
    K = len(cuts) - 1
    heavy = lens > exact_row_max
    if bool(heavy.any()):
        band[heavy[row_of]] = K - 1
    out = []
    for k in range(K):
        sel = band == k
        cnt = torch.bincount(row_of[sel], minlength=m)
        ptr = torch.zeros(m + 1, dtype=torch.int32, device=dev)
        ptr[1:] = torch.cumsum(cnt, 0).to(torch.int32)
        nk = int(ptr[-1].item()) if m else 0
        ck = torch.empty(nk + 8, dtype=torch.int32, device=dev)
        vk = torch.empty(nk + 8, dtype=torch.float64, device=dev)
        ck[:nk] = col[sel]
        vk[:nk] = val[sel]
        out.append(DeviceCsrArrays(m, arr.num_cols, nk, ptr, ck, vk))
    return out


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


_STAGING = {}
STAGING_BYTES = 32 << 20


def upload(a, dtype, device) -> torch.Tensor:
    """Host array -> new device tensor of `dtype` through two reused pinned
    staging buffers: the dtype conversion happens in the copy into pinned
    memory and overlaps the previous chunk's DMA (pageable copies of a user's
    numpy arrays run at a fraction of the PCIe rate)."""
    src = np.asarray(a)
    dt = np.dtype(dtype)
    n = int(src.shape[0])
    out = torch.empty(n, dtype=torch.from_numpy(np.zeros(0, dt)).dtype, device=device)
    if n == 0:
        return out
    if n * dt.itemsize <= (1 << 20):           # small: one pageable copy
        return out.copy_(torch.from_numpy(np.ascontiguousarray(src, dtype=dt)))
    key = (str(device),)
    bufs = _STAGING.get(key)
    if bufs is None:
        bufs = [(torch.empty(STAGING_BYTES, dtype=torch.uint8).pin_memory(), torch.cuda.Event()) for _ in range(2)]
        _STAGING[key] = bufs
    per = STAGING_BYTES // dt.itemsize
    stream = torch.cuda.current_stream(device)
    for k, lo in enumerate(range(0, n, per)):
        hi = min(n, lo + per)
        buf, ev = bufs[k & 1]
        ev.synchronize()                         # the DMA that last read this buffer is done
        view = buf[: (hi - lo) * dt.itemsize].numpy().view(dt)
        np.copyto(view, src[lo:hi], casting="unsafe")
        out[lo:hi].copy_(torch.from_numpy(view), non_blocking=True)
        ev.record(stream)
    return out


def upload_csr(A, device):
    """The user's CSR (row_offsets int64, col_indices -> int32, values f64)
    into HBM; the device setup's input (it needs no layout, so the solver
    starts it while the layout is computed)."""
    nnz = int(len(A.values))
    ptr = upload(A.row_offsets, np.int64, device)
    col = upload(A.col_indices, np.int32, device) if nnz else torch.zeros(1, dtype=torch.int32, device=device)
    val = upload(A.values, np.float64, device) if nnz else torch.zeros(1, dtype=torch.float64, device=device)
    return ptr, col, val


class DeviceSetup:
    """One-off device preprocessing through the C ABI (csrc/gridlp_setup.cu):
    the original CSR is uploaded once; every local block is then extracted
    (permuted, column-banded, rows sorted by column), transposed and laid
    out as SELL-32 on the device. Replaces the host permute/slice/transpose
    (partition.py:262-319, sparse_kernels.py:27-58)."""

    def __init__(self, problem, layout, device, preload=None):
        self.lib = native.load()
        self.device = device
        self.layout = layout
        A = problem.matrix
        m, n = int(A.num_rows), int(A.num_cols)
        if n >= 2 ** 31 - 1 or m >= 2 ** 31 - 1:
            raise ValueError("device setup needs < 2^31 rows and columns per matrix")
        nnz = int(np.asarray(A.row_offsets)[-1]) if m else 0       # (a scaled LP's values live on the device)
        self.nnz, self.n = nnz, n

        def t(a, dt):
            return upload(a, dt, device)

        t0 = time.perf_counter()
        self.src_ptr, self.src_col, self.src_val = preload if preload is not None else upload_csr(A, device)
        t1 = time.perf_counter()
        # the column permutation goes up once; its inverse is a device scatter
        self.col_perm = t(layout.perm.col_perm, np.int32) if n else torch.zeros(1, dtype=torch.int32, device=device)
        self.inv_col = torch.zeros(max(n, 1), dtype=torch.int32, device=device)
        if n:
            self.inv_col[self.col_perm.long()] = torch.arange(n, dtype=torch.int32, device=device)
        self.row_perm = t(layout.perm.row_perm, np.int64) if m else torch.zeros(1, dtype=torch.int64,
                                                                                 device=device)
        t2 = time.perf_counter()
        items = max(nnz, m + n) + 64
        segs = (m + n) + (m + n) // 32 + 64
        wsb = int(self.lib._lib.gridlp_setup_workspace_bytes(items, segs))
        self.ws = torch.empty(wsb, dtype=torch.uint8, device=device)
        self.ws_bytes = wsb
        self.times = {"setup_up_matrix_s": t1 - t0, "setup_up_perm_s": t2 - t1,
                      "setup_ws_s": time.perf_counter() - t2}
        self.h2d_bytes = sum(x.numel() * x.element_size()
                             for x in (self.src_ptr, self.src_col, self.src_val, self.col_perm, self.row_perm))

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

    def col_counts_device(self) -> torch.Tensor:
        """Entries per column of the uploaded original matrix (device int32)."""
        n = int(self.inv_col.numel()) if self.n else 0
        out = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        self.lib.call("gridlp_col_counts", self.src_col.data_ptr(), self.nnz, n, out.data_ptr(), self._stream())
        return out[:n]

    def col_counts(self) -> np.ndarray:
        """Entries per column of the uploaded original matrix (device
        histogram, host int64 result)."""
        n = int(self.inv_col.numel()) if self.n else 0
        out = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        self.lib.call("gridlp_col_counts", self.src_col.data_ptr(), self.nnz, n, out.data_ptr(), self._stream())
        return out[:n].cpu().numpy().astype(np.int64)

    def permute(self, a: DeviceCsrArrays, row_order: torch.Tensor | None,
                col_label: torch.Tensor | None) -> DeviceCsrArrays:
        """Rows gathered by row_order, columns relabelled by col_label (int32
        device tensors or None), entry order kept (gridlp_csr_permute)."""
        ptr = torch.empty(a.num_rows + 1, dtype=torch.int32, device=self.device)
        col = torch.empty(a.nnz + 8, dtype=torch.int32, device=self.device)
        val = torch.empty(a.nnz + 8, dtype=torch.float64, device=self.device)
        p = lambda t: t.data_ptr() if t is not None and t.numel() else None  # noqa: E731
        self.lib.call("gridlp_csr_permute", a.ptr.data_ptr(), a.col.data_ptr(), a.val.data_ptr(), a.num_rows,
                      p(row_order), p(col_label), ptr.data_ptr(), col.data_ptr(), val.data_ptr(), self.ws.data_ptr(),
                      self.ws_bytes, self._stream())
        return DeviceCsrArrays(a.num_rows, a.num_cols, a.nnz, ptr, col, val)

    def sell(self, a: DeviceCsrArrays, light_row_max: int) -> dict:
        """SELL-32 arrays built on the device (same as build_sell)."""
        dev, m = self.device, a.num_rows
        ns = (m + 31) // 32
        i32 = dict(dtype=torch.int32, device=dev)
        lane_info = torch.empty(max(ns * 32, 1), **i32)
        slice_off = torch.empty(ns + 1, dtype=torch.int64, device=self.device)
        rank_of = torch.empty(max(m, 1), **i32)
        long_rows = torch.empty(max(m, 1), **i32)
        long_ptr = torch.empty(m + 1, **i32)
        sizes = torch.zeros(3, dtype=torch.int64, device=dev)
        self.lib.call("gridlp_sell_plan", a.ptr.data_ptr(), m, light_row_max, lane_info.data_ptr(),
                      slice_off.data_ptr(), rank_of.data_ptr(), long_rows.data_ptr(), long_ptr.data_ptr(),
                      sizes.data_ptr(), self.ws.data_ptr(), self.ws_bytes, self._stream())
        total, nh, hnnz = (int(v) for v in sizes.cpu().tolist())
        sell_col = torch.empty(total + 8, **i32)
        sell_val = torch.empty(total + 8, dtype=torch.float64, device=dev)
        hcol = torch.empty(hnnz + 8, **i32)
        hval = torch.empty(hnnz + 8, dtype=torch.float64, device=dev)
        self.lib.call("gridlp_sell_fill", a.ptr.data_ptr(), a.col.data_ptr(), a.val.data_ptr(), m, light_row_max,
                      slice_off.data_ptr(), rank_of.data_ptr(), long_rows.data_ptr(), long_ptr.data_ptr(), nh,
                      sell_col.data_ptr(), sell_val.data_ptr(), total, hcol.data_ptr(), hval.data_ptr(),
                      self._stream())
        return dict(vals=sell_val, cols=sell_col, slice_off=slice_off, lane_info=lane_info,
                    num_slices=ns, long_rows=long_rows[:nh].clone() if nh else long_rows[:0],
                    long_ptr=long_ptr[: nh + 1].clone(), long_cols=hcol, long_vals=hval,
                    src_vals=a.val[: a.nnz])

    def release(self):
        for name in ("src_ptr", "src_col", "src_val", "col_perm", "inv_col", "row_perm", "ws"):
            setattr(self, name, None)


class BandSetup(DeviceSetup):
    """DeviceSetup for a band problem (synth.BandProblem): nothing is
    uploaded; block(i, j) is generated on the device by the problem's band
    generator, then transposed / permuted / laid out like any other block."""

    def __init__(self, problem, layout, device):
        self.lib = native.load()
        self.device = device
        self.layout = layout
        self.bands = problem.bands
        self.h2d_bytes = 0
        self.ws, self.ws_bytes = None, 0

    def _workspace(self, items: int, segs: int):
        need = int(self.lib._lib.gridlp_setup_workspace_bytes(items + 64, segs + 64))
        if need > self.ws_bytes:
            self.ws, self.ws_bytes = torch.empty(need, dtype=torch.uint8, device=self.device), need

    def block(self, i: int, j: int) -> DeviceCsrArrays:
        r0, r1 = self.layout.row_range(i)
        c0, c1 = self.layout.col_range(j)
        a = self.bands.block(r0, r1, c0, c1)
        self._workspace(a.nnz, max(r1 - r0, c1 - c0))
        return a

    def release(self):
        self.ws = None
