mkdir -p gpurun_out
python - <<'PY' > gpurun_out/e2e.log 2>&1
import time, sys, torch, json
sys.path.insert(0, ".")
from bench import make_problem
from paper_2601_07628_b200 import SolverConfig, solve
p = make_problem("cfg2")
for k in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    r = solve(p, SolverConfig(tolerance=1e-4, seed=0))
    torch.cuda.synchronize(); w = time.perf_counter() - t
    print(k, round(w, 3), r.status, r.iterations, {a: round(b, 4) for a, b in r.timings.items() if a.endswith("_s")}, flush=True)
PY
cat gpurun_out/e2e.log
