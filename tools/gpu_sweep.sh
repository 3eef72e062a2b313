# bench lines for a list of flag sets on one config: CFG, SETS ("tag:flags;tag:flags")
mkdir -p gpurun_out
CFG=${CFG:-cfg3}
IFS=';' read -ra ARR <<< "$SETS"
for item in "${ARR[@]}"; do
  tag=${item%%:*}; flags=${item#*:}
  timeout 900 python bench.py --config $CFG --steps ${STEPS:-10} --warmup 3 --no-e2e --no-cpu-baseline --no-spmv --no-extra $flags \
    > gpurun_out/sw_${CFG}_$tag.log 2>&1
  python - "gpurun_out/sw_${CFG}_$tag.log" "$CFG $tag" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k = d["kernels"]
    print(sys.argv[2], "us/iter", round(d["roofline"]["seconds_per_launch"] * 1e6, 1), "frac", round(d["roofline"]["frac"], 3),
          "K", {a: round(b["seconds"] * 1e6, 1) for a, b in k.items()}, "sm_mhz", d["clocks"].get("sm_mhz"))
except Exception as e:
    print(sys.argv[2], "parse failed", e); print(open(sys.argv[1]).read()[-1500:])
PY
done
