# row-class / internal-order sweep on the structured configs (bench lines, device time):
#   bash tools/sweep_layout.sh > gpurun_out/sweep_layout.txt
mkdir -p gpurun_out/sweep
run() {  # tag, args...
  local tag=$1; shift
  timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-spmv "$@" > gpurun_out/sweep/$tag.log 2>&1
  python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/sweep/{tag}.log").read().strip().splitlines()[-1])
    print(f"{tag:28s} {d['roofline']['seconds_per_launch'] * 1e6:9.1f} us/iter  frac {d['roofline']['frac']:.3f}  "
          f"K {({a: round(b['seconds'] * 1e6, 1) for a, b in d['kernels'].items()})}", flush=True)
except Exception as e:
    print(tag, "failed", e, open(f"gpurun_out/sweep/{tag}.log").read()[-800:])
PY
}
[ "$1" = "--defs-only" ] && return 0
for L in 128 256 512 1024; do
  run cfg4s_none_L$L --config cfg4s --permutation none --light-row-max $L
  run cfg4s_none_nat_L$L --config cfg4s --permutation none --light-row-max $L --natural-order
done
for L in 128 256 512; do
  run cfg3s_L$L --config cfg3s --light-row-max $L
  run cfg3s_nat_L$L --config cfg3s --light-row-max $L --natural-order
done
for L in 128 256 512; do
  run cfg4_none_L$L --config cfg4 --permutation none --light-row-max $L
  run cfg4_none_nat_L$L --config cfg4 --permutation none --light-row-max $L --natural-order
done
run cfg3_L128 --config cfg3
run cfg3_L256 --config cfg3 --light-row-max 256
run cfg3_nat_L128 --config cfg3 --natural-order
run cfg2_L256 --config cfg2 --light-row-max 256
run cfg2_nat --config cfg2 --natural-order
