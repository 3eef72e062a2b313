"""Interleaved A/B of kernel knobs (gridlp_set_tuning) on ONE engine in ONE
process: the same problem, the same box and clock state, variants
alternated rep by rep (the chunk graph is re-captured after each switch), so
box-to-box and run-to-run drift (±2-3 % between boxes) cancels.

    python tools/ab_variants.py --config cfg2 --key sell_variant --values 1 2 --reps 6
"""

import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2601_07628_b200 import SolverConfig, native  # noqa: E402
from paper_2601_07628_b200.api import prepare  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--key", default="sell_variant")
    ap.add_argument("--values", type=int, nargs="+", default=[1, 2])
    ap.add_argument("--reps", type=int, default=6)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--permutation", default=None)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    p = bench.make_problem(args.config)
    kw = dict(tolerance=1e-300, max_iterations=10**12, seed=0)
    if args.permutation:
        kw.update(permutation=args.permutation, partitioning="uniform")
    engine, layout, eta, omega, _ = prepare(p, SolverConfig(**kw), device=dev)
    engine.start(eta, omega)
    lib = native.load()
    old = lib.get_tuning(args.key)
    res = {v: [] for v in args.values}
    for rep in range(args.reps):
        for v in (args.values if rep % 2 == 0 else list(reversed(args.values))):
            lib.set_tuning(args.key, v)
            engine._graph = None          # re-capture with the new kernels
            for _ in range(2):
                engine.step()
            torch.cuda.synchronize()
            engine.iteration_events = []
            for _ in range(args.steps):
                engine.step()
            torch.cuda.synchronize()
            ev = engine.iteration_events
            engine.iteration_events = None
            t = sum(a.elapsed_time(b) for a, b, _ in ev) * 1e-3 / max(sum(n for _, _, n in ev), 1)
            res[v].append(t * 1e6)
    lib.set_tuning(args.key, old)
    out = {"config": args.config, "key": args.key,
           "us_per_iteration": {str(v): {"median": statistics.median(x), "all": [round(y, 2) for y in x]}
                                for v, x in res.items()}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
