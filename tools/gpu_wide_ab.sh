# GRIDLP_CSR_WIDE_CTAS launch hint: parity tests + interleaved A/B (tuning "wide_ctas" 1 = honour the hint, 0 = ignore)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_codec.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_wide.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_wide.log
timeout 900 python tools/ab_variants.py --config cfg4 --permutation none --key wide_ctas --values 0 1 --reps 4 --steps 2 > gpurun_out/ab_wide_cfg4.json 2> gpurun_out/ab_wide_cfg4.err; echo "cfg4 rc=$?"; cat gpurun_out/ab_wide_cfg4.json
timeout 900 python tools/ab_variants.py --config cfg2 --key wide_ctas --values 0 1 --reps 4 > gpurun_out/ab_wide_cfg2.json 2> gpurun_out/ab_wide_cfg2.err; echo "cfg2 rc=$?"; cat gpurun_out/ab_wide_cfg2.json
