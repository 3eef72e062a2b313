# interleaved A/B of sell_variant on cfg2 / cfg3 / cfg4 (tools/ab_variants.py)
mkdir -p gpurun_out
timeout 900 python tools/ab_variants.py --config cfg2 --values 1 2 --reps 8 > gpurun_out/ab_cfg2.json 2> gpurun_out/ab_cfg2.err; echo "cfg2 rc=$?"; cat gpurun_out/ab_cfg2.json
timeout 900 python tools/ab_variants.py --config cfg3 --values 1 2 --reps 4 --steps 2 > gpurun_out/ab_cfg3.json 2> gpurun_out/ab_cfg3.err; echo "cfg3 rc=$?"; cat gpurun_out/ab_cfg3.json
timeout 900 python tools/ab_variants.py --config cfg4 --permutation none --values 1 2 --reps 4 --steps 2 > gpurun_out/ab_cfg4.json 2> gpurun_out/ab_cfg4.err; echo "cfg4 rc=$?"; cat gpurun_out/ab_cfg4.json
