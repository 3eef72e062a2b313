mkdir -p gpurun_out
./tools/microbench > gpurun_out/microbench.log 2>&1; echo "mb rc=$?"
cat gpurun_out/microbench.log
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:tile_kernel<.*OpDual' -s 200 -c 1 -o gpurun_out/prof_v1_dual python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --variant 1 > gpurun_out/ncu_v1.log 2>&1; echo "ncu rc=$?"
