# kernel-variant sweep: GPU parity tests on the default variant, then bench
# lines per sell_variant / chain_products on the given configs.
# env: CFGS (default "cfg2 cfg3"), VARIANTS (default "0 1 2 3 4"), PYTEST_K
mkdir -p gpurun_out
if [ -n "${PYTEST_K:-}" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$PYTEST_K" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
  tail -5 gpurun_out/pytest_gpu.log
fi
for cfg in ${CFGS:-cfg2 cfg3}; do
  for v in ${VARIANTS:-0 1 2 3 4}; do
    for ch in ${CHAINS:-1}; do
      tag=${cfg}_v${v}_c${ch}
      timeout 900 python bench.py --config $cfg --steps ${STEPS:-10} --warmup 3 --no-e2e --no-cpu-baseline --no-spmv --no-extra \
        --tuning sell_variant=$v --tuning chain_products=$ch $EXTRA > gpurun_out/var_$tag.log 2>&1
      python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/var_{tag}.log").read().strip().splitlines()[-1]); k = d["kernels"]
    print(tag, "us/iter", round(d["roofline"]["seconds_per_launch"] * 1e6, 1), "frac", round(d["roofline"]["frac"], 3),
          "K", {a: round(b["seconds"] * 1e6, 1) for a, b in k.items()}, "sm_mhz", d["clocks"].get("sm_mhz"))
except Exception as e:
    print(tag, "parse failed", e); print(open(f"gpurun_out/var_{tag}.log").read()[-1500:])
PY
    done
  done
done
