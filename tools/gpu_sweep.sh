mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "Products" > gpurun_out/pytest_products.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_products.log
for V in ${@:-6 7 8 5}; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --variant $V > gpurun_out/bench_v$V.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_v$V.log').read().strip().splitlines()[-1]); k=d['kernels']; print('v$V', round(d['value']), 'it/s', round(d['roofline']['seconds_per_launch']*1e6,1), 'us/iter frac', round(d['roofline']['frac'],3), 'K1', round(k['K1']['seconds']*1e6,1), 'K2', round(k['K2']['seconds']*1e6,1))" || tail -5 gpurun_out/bench_v$V.log
done
