mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_parity.py tests/test_gpu_variants.py -q -x -p no:cacheprovider > gpurun_out/pytest_codec.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_codec.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-spmv --no-extra > gpurun_out/bench_cfg2_codec.log 2>&1; echo "bench cfg2 rc=$?"; tail -1 gpurun_out/bench_cfg2_codec.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg2', r['seconds_per_launch']*1e6, r['frac'], d['clocks'])"
TAG=cfg4_auto bash tools/gpu_cfg.sh cfg4 --permutation none --no-e2e --no-cpu-baseline --no-spmv --no-extra
TAG=cfg4_f64 bash tools/gpu_cfg.sh cfg4 --permutation none --no-e2e --no-cpu-baseline --no-spmv --no-extra --value-codec f64
