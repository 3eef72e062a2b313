"""The reference algorithm's own time-to-1e-4 on cfg2, on this host: the
CPU oracle (oracle/pdhg_oracle.py — bit-for-bit the reference's
reference_solve) run to completion on one core, as the e2e counterpart of
the bench's GPU solve. Minutes of CPU; run on the GPU box to compare with
the GPU e2e in the same environment."""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from threadpoolctl import threadpool_limits  # noqa: E402

from bench import make_problem  # noqa: E402
from oracle import pdhg_oracle  # noqa: E402

p = make_problem(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
with threadpool_limits(1):
    t0 = time.perf_counter()
    r = pdhg_oracle.oracle_solve(p, tolerance=1e-4, seed=0)
    wall = time.perf_counter() - t0
print(json.dumps({"what": "reference algorithm (CPU oracle, 1 core) time-to-1e-4", "config": sys.argv[1:] or ["cfg2"],
                  "seconds": wall, "status": r.status, "iterations": r.iterations, "restarts": r.restarts,
                  "objective": r.objective, "cpu": os.cpu_count()}), flush=True)
