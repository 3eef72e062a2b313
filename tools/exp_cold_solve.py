"""Cold vs warm complete solves in one fresh process (the first solve pays
CUDA context / module / allocator warm-up): per-phase timings of solves 1-3.

    python tools/exp_cold_solve.py [cfg2]
"""

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2601_07628_b200 import SolverConfig, solve  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    p = bench.make_problem(args[0] if args else "cfg2")
    torch.cuda.synchronize()
    if "--warmup" in sys.argv:
        from paper_2601_07628_b200 import warmup

        t0 = time.perf_counter()
        warmup()
        print(f"warmup() {time.perf_counter() - t0:.3f}s", flush=True)
    for k in range(3):
        t0 = time.perf_counter()
        r = solve(p, SolverConfig(tolerance=1e-4, seed=0))
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        keys = ("layout_s", "setup_blocks_s", "power_s", "main_loop_s")
        print(f"solve {k + 1}: {wall:.3f}s", {kk: round(r.timings.get(kk, 0.0), 4) for kk in keys}, flush=True)


if __name__ == "__main__":
    main()
