# GPU suite + default bench (no e2e/cpu legs unless FULL=1)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log | grep -E "passed|failed|Error|error" | head -10
if [ "${FULL:-0}" = 1 ]; then EXTRA=""; else EXTRA="--no-e2e --no-cpu-baseline --no-spmv --no-extra"; fi
timeout 900 python bench.py --steps 10 --warmup 3 $EXTRA > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
try:
    d = json.loads(open("gpurun_out/bench.log").read().strip().splitlines()[-1]); k = d["kernels"]
    print("value", round(d["value"]), "it/s; us/iter", round(d["roofline"]["seconds_per_launch"] * 1e6, 1), "frac", round(d["roofline"]["frac"], 3),
          "K1", round(k["K1"]["seconds"] * 1e6, 1), "K2", round(k["K2"]["seconds"] * 1e6, 1), "e2e", (d.get("e2e") or {}).get("time_to_tol_s"))
except Exception as e:
    print("bench parse failed", e); print(open("gpurun_out/bench.log").read()[-2000:])
PY
