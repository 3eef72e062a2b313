"""Per-step timeline of one solve's main loop (cfg2 by default): host wall
time of each engine.step() (64 iterations + KKT pass) next to the device
time of its graph replays, to locate main-loop time that is not kernel time.

    python tools/e2e_steps.py [--config cfg2]
"""

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    args = ap.parse_args()
    import torch

    from paper_2601_07628_b200 import SolverConfig, solve
    from paper_2601_07628_b200.api import prepare

    p = bench.make_problem(args.config)
    solve(p, SolverConfig(tolerance=1e-4, seed=0))        # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng, lay, eta, omega, tim = prepare(p, SolverConfig(tolerance=1e-4, seed=0))
    torch.cuda.synchronize()
    t_prep = time.perf_counter() - t0
    eng.start(eta, omega)
    eng.iteration_events = []
    rows = []
    t_loop = time.perf_counter()
    while True:
        a = time.perf_counter()
        done = eng.step()
        b = time.perf_counter()
        rows.append(b - a)
        if done:
            break
    out = eng.finish()
    torch.cuda.synchronize()
    t_end = time.perf_counter()
    dev = [x.elapsed_time(y) * 1e-3 for x, y, _ in eng.iteration_events]
    print(json.dumps({"prepare_s": t_prep, "loop_s": t_end - t_loop, "steps": len(rows),
                      "step_wall_s_first5": rows[:5], "step_wall_s_median": sorted(rows)[len(rows) // 2],
                      "device_iter_s_first5": dev[:5], "device_iter_s_median": sorted(dev)[len(dev) // 2] if dev else None,
                      "sum_step_wall_s": sum(rows), "sum_device_iter_s": sum(dev), "status": out["status"],
                      "iterations": out["iterations"]}))


if __name__ == "__main__":
    main()
