"""Time each host->HBM upload of the device setup for one config (the e2e
setup_upload_s breakdown).

    python tools/exp_setup_upload.py [cfg2]
"""

import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_2601_07628_b200 import blocks  # noqa: E402
from paper_2601_07628_b200.layout import build_layout  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    p = bench.make_problem(name)
    A = p.matrix
    dev = torch.device("cuda", 0)
    lay = build_layout(p, n_procs=1, block_size=64, seed=0, permutation="block_random", partitioning="nnz")
    print("threads", blocks.UPLOAD_THREADS, {k: (getattr(A, k).dtype, getattr(A, k).nbytes >> 20)
                                             for k in ("row_offsets", "col_indices", "values")})
    for rep in range(3):
        for nm, a, dt in (("ptr", A.row_offsets, np.int64), ("col", A.col_indices, np.int32),
                          ("val", A.values, np.float64), ("col_perm", lay.perm.col_perm, np.int32),
                          ("row_perm", lay.perm.row_perm, np.int64), ("obj", p.objective, np.float64)):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            blocks.upload(a, dt, dev)
            torch.cuda.synchronize()
            t = time.perf_counter() - t0
            print(f"rep{rep} {nm:9s} {np.asarray(a).dtype}->{np.dtype(dt)} {np.asarray(a).nbytes / 2**20:7.1f} MiB "
                  f"{t * 1e3:7.2f} ms {np.asarray(a).nbytes / t / 1e9:6.2f} GB/s", flush=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s = blocks.DeviceSetup(p, lay, dev)
        torch.cuda.synchronize()
        print(f"rep{rep} DeviceSetup {1e3 * (time.perf_counter() - t0):.2f} ms h2d {s.h2d_bytes >> 20} MiB")
        del s


if __name__ == "__main__":
    main()
