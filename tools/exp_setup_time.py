"""Time solve() setup phases on cfg2 twice (second = warm process)."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import make_problem  # noqa: E402
from paper_2601_07628_b200 import SolverConfig, solve  # noqa: E402

p = make_problem(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = solve(p, SolverConfig(tolerance=1e-4, seed=0))
    torch.cuda.synchronize()
    w = time.perf_counter() - t0
    print(f"rep {rep}: {w:.3f}s {r.status} it={r.iterations}",
          {k: round(v, 4) for k, v in r.timings.items() if k.endswith("_s")}, flush=True)
