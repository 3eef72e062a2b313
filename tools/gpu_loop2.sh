mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_device_loop.py -q -x -p no:cacheprovider > gpurun_out/pytest_loop.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_loop.log
for flag in "" "--no-device-loop" "" "--no-device-loop"; do
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-spmv --no-e2e --no-extra $flag > gpurun_out/bench_loop2.log 2>&1; echo "bench rc=$? $flag"
tail -1 gpurun_out/bench_loop2.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('value', round(d['value']), 'ms/step', round(d['ms_per_step'],3), 'us/iter', round(d['roofline']['seconds_per_launch']*1e6,1), 'frac', round(d['roofline']['frac'],3), 'launches', d['gpu_launches'], d['config']['main_loop'][:6], d['clocks']['reasons'])"
done
