# device-side loop: parity tests + golden solves + e2e / cfg1 numbers
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_device_loop.py tests/test_gpu_parity.py tests/test_gpu_solver_api.py tests/test_gpu_acceptance.py tests/test_gpu_codec.py -q -x -p no:cacheprovider > gpurun_out/pytest_loop.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_loop.log | grep -E "passed|failed|Error|assert" | head -12
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-spmv > gpurun_out/bench_loop.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_loop.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; c=d['extra_configs']['cfg1_latency']
print('value', round(d['value']), 'us/iter', round(d['roofline']['seconds_per_launch']*1e6,1), 'e2e', e['time_to_tol_s'], e['runs_s'], e['status'], e['iterations'], 'cfg1', c['time_to_tol_s'], c['runs_s'], c['iterations'], 'launches', d['gpu_launches'])"
