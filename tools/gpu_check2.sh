mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_device_loop.py tests/test_gpu_bounds.py tests/test_gpu_codec.py -q -x -p no:cacheprovider > gpurun_out/pytest_check2.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_check2.log
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_check2.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_check2.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; e=d['e2e']; x=d['extra_configs']
print('value', round(d['value']), 'us/iter', round(r['seconds_per_launch']*1e6,1), 'frac', round(r['frac'],3), d['clocks'])
print('e2e', e['time_to_tol_s'], e['runs_s'], e['status'], e['iterations'])
print('cfg1', x['cfg1_latency']['time_to_tol_s'], x['cfg1_latency']['runs_s'])
print('cfg3', round(x['cfg3']['us_per_iteration'],1), round(x['cfg3']['frac'],3))"
