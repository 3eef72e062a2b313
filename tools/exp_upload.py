"""Host->HBM upload strategies for the e2e setup (the user's pageable numpy
arrays): pinned staging with 1..T copy threads, chunk size, and in-place
page-locking (cudaHostRegister). Prints GB/s per strategy.

    python tools/exp_upload.py
"""

import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def staged(src, dt, dev, threads, chunk, nbuf, pool):
    n = src.shape[0]
    out = torch.empty(n, dtype=torch.from_numpy(np.zeros(0, dt)).dtype, device=dev)
    bufs = staged.bufs.get((chunk, nbuf))
    if bufs is None:
        bufs = [(torch.empty(chunk, dtype=torch.uint8).pin_memory(), torch.cuda.Event()) for _ in range(nbuf)]
        staged.bufs[(chunk, nbuf)] = bufs
    per = chunk // dt.itemsize
    stream = torch.cuda.current_stream(dev)
    for k, lo in enumerate(range(0, n, per)):
        hi = min(n, lo + per)
        buf, ev = bufs[k % nbuf]
        ev.synchronize()
        view = buf[: (hi - lo) * dt.itemsize].numpy().view(dt)
        if threads == 1:
            np.copyto(view, src[lo:hi], casting="unsafe")
        else:
            step = -(-(hi - lo) // threads)
            list(pool.map(lambda t: np.copyto(view[t * step:(t + 1) * step], src[lo + t * step:min(hi, lo + (t + 1) * step)],
                                              casting="unsafe"), range(threads)))
        out[lo:hi].copy_(torch.from_numpy(view), non_blocking=True)
        ev.record(stream)
    return out


staged.bufs = {}


def registered(src, dt, dev):
    assert src.dtype == dt
    cud = torch.cuda.cudart()
    ptr, nb = src.ctypes.data, src.nbytes
    t0 = time.perf_counter()
    r = cud.cudaHostRegister(ptr, nb, 0)
    t1 = time.perf_counter()
    out = torch.empty(src.shape[0], dtype=torch.from_numpy(np.zeros(0, dt)).dtype, device=dev)
    out.copy_(torch.from_numpy(src), non_blocking=True)
    torch.cuda.current_stream(dev).synchronize()
    t2 = time.perf_counter()
    cud.cudaHostUnregister(ptr)
    t3 = time.perf_counter()
    return out, (r, t1 - t0, t2 - t1, t3 - t2)


def main():
    dev = torch.device("cuda", 0)
    print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
    rng = np.random.default_rng(0)
    vals = rng.standard_normal(20_000_000)
    cols = rng.integers(0, 2_000_000, 20_000_000).astype(np.int32)
    cols64 = cols.astype(np.int64)
    pool = ThreadPoolExecutor(16)
    cases = [("f64 160MB", vals, np.float64), ("i32 80MB", cols, np.int32), ("i64->i32", cols64, np.int32)]
    for name, src, dt in cases:
        for threads in (1, 2, 4, 8):
            for chunk, nbuf in ((32 << 20, 2), (8 << 20, 4), (64 << 20, 2)):
                best = 1e9
                for _ in range(4):
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    staged(src, np.dtype(dt), dev, threads, chunk, nbuf, pool)
                    torch.cuda.synchronize()
                    best = min(best, time.perf_counter() - t0)
                print(f"{name:10s} staged T={threads} chunk={chunk >> 20}MB x{nbuf}: {best * 1e3:7.2f} ms "
                      f"{src.nbytes / best / 1e9:6.2f} GB/s(src)", flush=True)
        if src.dtype == dt:
            for _ in range(2):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                _, parts = registered(src, np.dtype(dt), dev)
                t = time.perf_counter() - t0
                print(f"{name:10s} hostRegister: {t * 1e3:7.2f} ms (register/copy/unregister {parts}) "
                      f"{src.nbytes / t / 1e9:6.2f} GB/s", flush=True)
    # the pageable baseline
    for name, src, dt in cases[:1]:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        torch.from_numpy(src).to(dev)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        print(f"{name:10s} pageable .to(): {t * 1e3:7.2f} ms {src.nbytes / t / 1e9:6.2f} GB/s")


if __name__ == "__main__":
    main()
