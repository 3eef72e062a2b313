"""µs per PDHG iteration of small LPs (the launch-bound regime of BASELINE
configs[0]): the persistent cooperative launch, the CUDA-graph path (kernel
per product, chained) and the cluster launch (falls back to the graph path
when the LP does not fit), and time to 1e-4 for cfg1 each way.

    python tools/persistent_sweep.py
"""

import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def per_iter(p, over, steps=20):
    import torch

    from paper_2601_07628_b200 import SolverConfig
    from paper_2601_07628_b200.api import prepare

    eng, lay, eta, omega, _ = prepare(p, SolverConfig(tolerance=1e-300, max_iterations=10**12, seed=0),
                                      engine_overrides=over)
    eng.start(eta, omega)
    for _ in range(3):
        eng.step()
    torch.cuda.synchronize()
    eng.iteration_events = []
    for _ in range(steps):
        eng.step()
    torch.cuda.synchronize()
    ev = eng.iteration_events
    return sum(a.elapsed_time(b) for a, b, _ in ev) * 1e3 / sum(n for _, _, n in ev)


def main():
    from paper_2601_07628_b200 import GeneratorSpec, SolverConfig, generate
    from paper_2601_07628_b200.api import _solve

    for m, n, nnz in ((2000, 4000, 20000), (6000, 12000, 60000), (20000, 40000, 200000), (60000, 120000, 600000)):
        p = generate(GeneratorSpec(kind="uniform_random", num_rows=m, num_cols=n, nnz_target=nnz,
                                   inequality_fraction=0.3, seed=0))
        on = per_iter(p, {"persistent_max_nnz": 1 << 30, "cluster_small": False})
        off = per_iter(p, {"persistent_max_nnz": 0, "cluster_small": False})
        cl = per_iter(p, {"persistent_max_nnz": 0, "cluster_small": True})
        print(json.dumps({"m": m, "n": n, "nnz": nnz, "persistent_us_per_iter": on, "graph_us_per_iter": off,
                          "cluster_or_fallback_us_per_iter": cl}), flush=True)
    p = generate(GeneratorSpec(kind="uniform_random", num_rows=2000, num_cols=4000, nnz_target=20000,
                               inequality_fraction=0.3, seed=0))
    for name, over in (("persistent", {"persistent_max_nnz": 1 << 30, "cluster_small": False}),
                       ("graph", {"persistent_max_nnz": 0, "cluster_small": False}),
                       ("cluster", {"persistent_max_nnz": 0, "cluster_small": True})):
        _solve(p, SolverConfig(tolerance=1e-4, seed=0), engine_overrides=over)
        walls = []
        for _ in range(3):
            t0 = time.perf_counter()
            r = _solve(p, SolverConfig(tolerance=1e-4, seed=0), engine_overrides=over)
            walls.append(time.perf_counter() - t0)
        print(json.dumps({"cfg1": name, "time_to_tol_s": sorted(walls)[1], "iterations": r.iterations,
                          "status": r.status, "objective": r.objective}), flush=True)


if __name__ == "__main__":
    main()
