"""Reference-algorithm CPU throughput on the §8f configs (SURVEY §8d CPU
timing plan, item 3): main-loop iterations/s of the CPU oracle
(oracle/pdhg_oracle.py, the reference's algorithm with scipy csr_matvec) on
the GPU box's host — 1 thread on a 1x1 grid, and one thread per block on the
grid select_grid picks for the host's cores (the reference's threads
executor). The problem comes from the device generators, is copied to host
arrays and the GPU is released before the CPU part; an address-space limit
keeps a too-large config from taking the box's memory (MemoryError instead).

    python tools/cpu_configs.py cfg3 cfg4 [--iters 2]
"""

import argparse
import gc
import json
import os
import resource
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def _meminfo(key):
    with open("/proc/meminfo") as f:
        for line in f:
            if line.startswith(key + ":"):
                return int(line.split()[1]) * 1024
    return 0


def _vmsize():
    with open("/proc/self/status") as f:
        for line in f:
            if line.startswith("VmSize:"):
                return int(line.split()[1]) * 1024
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--mem-frac", type=float, default=0.5, help="address-space budget as a share of MemAvailable")
    args = ap.parse_args()
    import torch

    import bench
    from oracle import pdhg_oracle
    from paper_2601_07628_b200 import select_grid

    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except ImportError:  # pragma: no cover
        pass
    avail = _meminfo("MemAvailable")
    print(json.dumps({"cpus": os.cpu_count(), "mem_available_gb": avail / 2**30,
                      "mem_total_gb": _meminfo("MemTotal") / 2**30}), flush=True)
    budget = int(args.mem_frac * avail)
    limit_set = False
    for name in args.configs:
        t0 = time.perf_counter()
        p = bench.make_problem(name)
        gen_s = time.perf_counter() - t0
        torch.cuda.empty_cache()
        if not limit_set:
            soft, hard = resource.getrlimit(resource.RLIMIT_AS)
            resource.setrlimit(resource.RLIMIT_AS, (_vmsize() + budget, hard))
            limit_set = True
        threads = max(1, min(os.cpu_count() or 1, 32))
        g = select_grid(p.num_constraints, p.num_variables, threads)
        out = {"config": name, "m": p.num_constraints, "n": p.num_variables, "nnz": int(p.matrix.nnz),
               "generate_s": gen_s}
        for label, grid, th in (("1thread_1x1", (1, 1), 1), (f"{threads}threads", (g.rows, g.cols), g.rows * g.cols)):
            try:
                r = pdhg_oracle.iteration_rate(p, args.iters, grid=grid, threads=th)
                out[label] = r
            except MemoryError as e:
                out[label] = {"error": f"MemoryError under the {budget / 2**30:.0f} GiB budget: {e}"}
            gc.collect()
            print(json.dumps(out), flush=True)
        del p
        gc.collect()


if __name__ == "__main__":
    main()
