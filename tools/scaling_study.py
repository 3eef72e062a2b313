"""Scaled vs unscaled time-to-tolerance on a device-generated config
(SolverConfig.scaling, north-star item 4): status, iterations, restarts, the
original-LP KKT report, scaling time and wall, one JSON line per run.

    python tools/scaling_study.py cfg3 --tol 1e-4 --max-iter 20000
"""

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--tol", type=float, default=1e-4)
    ap.add_argument("--max-iter", type=int, default=20000)
    ap.add_argument("--modes", default="none,ruiz+pock_chambolle")
    ap.add_argument("--permutation", default=None)
    args = ap.parse_args()
    import torch

    from paper_2601_07628_b200 import SolverConfig, solve

    p = bench.make_problem(args.config)
    for mode in args.modes.split(","):
        kw = dict(tolerance=args.tol, max_iterations=args.max_iter, seed=0, scaling=mode)
        if args.permutation:
            kw["permutation"] = args.permutation
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = solve(p, SolverConfig(**kw))
        wall = time.perf_counter() - t0
        print(json.dumps({"config": args.config, "scaling": mode, "status": r.status, "iterations": r.iterations,
                          "restarts": r.restarts, "objective": r.objective, "kkt": r.report.as_dict(),
                          "wall_s": wall, "scaling_s": (r.timings or {}).get("scaling_s"),
                          "main_loop_s": (r.timings or {}).get("main_loop_s")}), flush=True)


if __name__ == "__main__":
    main()
