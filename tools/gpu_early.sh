# sell_variant 2 (epilogue operands requested before the row's gathers) vs 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_variants.py tests/test_gpu_codec.py -q -x -p no:cacheprovider > gpurun_out/pytest_early.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_early.log
for v in 1 2 1 2; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-spmv --no-extra --tuning sell_variant=$v > gpurun_out/bench_cfg2_v$v.log 2>&1
  tail -1 gpurun_out/bench_cfg2_v$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; k=d['kernels']; print('cfg2 v$v', round(r['seconds_per_launch']*1e6,1), round(r['frac'],3), 'K1', round(k['K1']['seconds']*1e6,1), 'K2', round(k['K2']['seconds']*1e6,1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
for v in 1 2; do TAG=cfg4_v$v bash tools/gpu_cfg.sh cfg4 --permutation none --no-e2e --no-cpu-baseline --no-spmv --no-extra --tuning sell_variant=$v | tail -1; done
for v in 1 2; do TAG=cfg3_v$v bash tools/gpu_cfg.sh cfg3 --no-e2e --no-cpu-baseline --no-spmv --no-extra --tuning sell_variant=$v | tail -1; done
