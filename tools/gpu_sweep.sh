# product-kernel A/B: parity of all variants, then bench lines per "variant:l2persist"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "Products" > gpurun_out/pytest_products.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_products.log
for VP in ${@:-9:0 9:1 11:0 11:1 12:0 12:1}; do
  V=${VP%%:*}; P=${VP##*:}
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --variant $V --l2-persist $P > gpurun_out/bench_v${V}_p$P.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_v${V}_p$P.log').read().strip().splitlines()[-1]); k=d['kernels']; print('v$V p$P', round(d['value']), 'it/s', round(d['roofline']['seconds_per_launch']*1e6,1), 'us/iter frac', round(d['roofline']['frac'],3), 'K1', round(k['K1']['seconds']*1e6,1), 'K2', round(k['K2']['seconds']*1e6,1), 'sm', d['clocks']['sm_mhz'])" || tail -5 gpurun_out/bench_v${V}_p$P.log
done
