# bench lines for the device-generated configs: tools/gpu_cfg.sh CFG [extra bench args...]
mkdir -p gpurun_out
CFG=$1; shift
TAG=${TAG:-$CFG}
timeout ${TMO:-1500} python bench.py --config $CFG --steps ${STEPS:-5} --warmup 3 "$@" > gpurun_out/bench_$TAG.log 2>&1; echo "bench $TAG rc=$?"
grep "^\[bench\]" gpurun_out/bench_$TAG.log | tail -3
python - "$TAG" <<'PY'
import json, sys
tag = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/bench_{tag}.log").read().strip().splitlines()[-1]); k = d["kernels"]
    print(tag, "value", round(d["value"], 1), "it/s; us/iter", round(d["roofline"]["seconds_per_launch"] * 1e6, 1), "frac", round(d["roofline"]["frac"], 3),
          "req frac", round(d["roofline"]["request_bound"]["frac"], 3), "K", {a: round(b["seconds"] * 1e6, 1) for a, b in k.items()},
          "balance", d["config"].get("block_nnz_max_over_mean"), "e2e", (d.get("e2e") or {}).get("time_to_tol_s"), (d.get("e2e") or {}).get("status"))
except Exception as e:
    print("parse failed", e); print(open(f"gpurun_out/bench_{tag}.log").read()[-3000:])
PY
