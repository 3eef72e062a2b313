# quick GPU check after a kernel change: parity/variant/codec/bounds tests + cfg2 and cfg4 bench lines
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_codec.py tests/test_gpu_bounds.py tests/test_gpu_sanitizer.py -q -x -p no:cacheprovider -rs > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_quick.log
for v in 2 1; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-spmv --no-extra --tuning sell_variant=$v > gpurun_out/bench_q_v$v.log 2>&1
  tail -1 gpurun_out/bench_q_v$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; k=d['kernels']; print('cfg2 v$v', round(r['seconds_per_launch']*1e6,1), round(r['frac'],3), 'K1', round(k['K1']['seconds']*1e6,1), 'K2', round(k['K2']['seconds']*1e6,1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
TAG=cfg4_q bash tools/gpu_cfg.sh cfg4 --permutation none --no-e2e --no-cpu-baseline --no-spmv --no-extra | tail -1
