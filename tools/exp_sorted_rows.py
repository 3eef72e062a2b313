"""Experiment: product time with rows in natural order vs rows sorted by
length (descending) — what a length-sorted internal row order would buy.
Also columns relabelled by degree (heavy first) for gather locality."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import make_problem  # noqa: E402
from paper_2601_07628_b200.blocks import DeviceCsr, HostCsr, transpose  # noqa: E402
from paper_2601_07628_b200.ops import CudaOps, Fused  # noqa: E402

dev = torch.device("cuda", 0)
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
p = make_problem(cfg)
M = p.matrix
h = HostCsr(M.num_rows, M.num_cols, np.asarray(M.row_offsets, np.int64), np.asarray(M.col_indices, np.int64),
            np.asarray(M.values))


def permute_rows(a: HostCsr, order):
    lens = np.diff(a.ptr)[order]
    ptr = np.concatenate([[0], np.cumsum(lens)])
    src = np.repeat(a.ptr[:-1][order] - ptr[:-1], lens) + np.arange(ptr[-1])
    return HostCsr(a.num_rows, a.num_cols, ptr, a.col[src], a.val[src])


def relabel_cols(a: HostCsr, newlabel):
    return HostCsr(a.num_rows, a.num_cols, a.ptr, newlabel[a.col], a.val)


def timeit(A, n):
    ops = CudaOps(dev, A.slots() + 8, 1)
    x = torch.randn(n, dtype=torch.float64, device=dev)
    out = torch.empty(A.num_rows, dtype=torch.float64, device=dev)
    for _ in range(3):
        ops.store(Fused(A, x), out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ops.store(Fused(A, x), out)
        b.record()
        ts.append((a, b))
    torch.cuda.synchronize()
    return sorted(x.elapsed_time(y) for x, y in ts)[10] * 1e3


for name, a in (("A", h), ("AT", transpose(h))):
    lens = np.diff(a.ptr)
    order = np.argsort(-lens, kind="stable")
    col_deg = np.bincount(a.col, minlength=a.num_cols)
    colorder = np.argsort(-col_deg, kind="stable")
    newlabel = np.empty_like(colorder)
    newlabel[colorder] = np.arange(a.num_cols)
    base = timeit(DeviceCsr(a, dev), a.num_cols)
    srt = timeit(DeviceCsr(permute_rows(a, order), dev), a.num_cols)
    both = timeit(DeviceCsr(relabel_cols(permute_rows(a, order), newlabel), dev), a.num_cols)
    print(f"{cfg} {name}: natural {base:.1f} us | rows sorted by length {srt:.1f} us | + cols by degree {both:.1f} us",
          flush=True)
