"""Full-size planted LP (bench.py CONFIGS["cfg5s"]: 12.5M x 20M, ~400M nnz,
generated block by block on the device as a BandProblem) solved through
solve() on one B200 to a relative KKT tolerance, against its analytic
optimum c·x* (sequential host dot of the device-generated c and x*).

    python tools/planted_full.py [--tol 1e-6] [--max-it 60000] [--name cfg5s]
"""

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2601_07628_b200 import SolverConfig, solve, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--name", default="cfg5s")
    ap.add_argument("--tol", type=float, default=1e-6)
    ap.add_argument("--max-it", type=int, default=60000)
    args = ap.parse_args()
    spec = dict(bench.CONFIGS[args.name])
    spec.pop("gen")
    dev = torch.device("cuda", 0)
    bands = synth.PlantedBands(synth.PlantedSpec(**spec), dev)
    c, _, _, x_star = bands.col_data(0, spec["num_cols"])
    star = float(np.dot(c.cpu().numpy(), x_star.cpu().numpy()))
    del c, x_star
    torch.cuda.empty_cache()
    prob = synth.BandProblem(bands, args.name)
    t0 = time.perf_counter()
    r = solve(prob, SolverConfig(tolerance=args.tol, seed=0, permutation="none", partitioning="uniform",
                                 max_iterations=args.max_it))
    wall = time.perf_counter() - t0
    print(json.dumps({"config": args.name, "tolerance": args.tol, "status": r.status, "iterations": r.iterations,
                      "restarts": r.restarts, "objective": r.objective, "planted_optimum": star,
                      "rel_err": abs(r.objective - star) / (1.0 + abs(star)), "kkt": r.report.as_dict(),
                      "wall_s": wall, "nnz": r.layout.get("total_nnz"),
                      "main_loop_s": (r.timings or {}).get("main_loop_s")}))


if __name__ == "__main__":
    main()
