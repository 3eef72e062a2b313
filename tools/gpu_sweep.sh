mkdir -p gpurun_out
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -3 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
for cfg in "0 2048" "0 1024" "0 4096" "1 2048" "1 4096"; do
  set -- $cfg
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --variant $1 --tile-cap $2 > gpurun_out/bench_v$1_c$2.log 2>&1
  echo "variant $1 cap $2 rc=$?"
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_v$1_c$2.log').read().strip().splitlines()[-1]); print('v$1 c$2', round(d['value']), 'it/s', d['roofline']['seconds_per_launch']*1e6, 'us/iter frac', round(d['roofline']['frac'],3), d['kernels'])" || tail -20 gpurun_out/bench_v$1_c$2.log
done
