mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_variants.py tests/test_gpu_nccl.py -q -x -p no:cacheprovider > gpurun_out/pytest_wide2.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_wide2.log
timeout 900 python tools/ab_variants.py --config cfg4 --permutation none --key wide_ctas --values 1 2 --reps 4 --steps 2 > gpurun_out/ab_wide2_cfg4.json 2> gpurun_out/ab_wide2_cfg4.err; echo "cfg4 rc=$?"; cat gpurun_out/ab_wide2_cfg4.json
