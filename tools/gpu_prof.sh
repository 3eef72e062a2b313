mkdir -p gpurun_out
V=${1:-5}
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:tile_kernel<.*OpDual' -s 30 -c 1 -o gpurun_out/prof_v${V}_dual python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --variant $V > gpurun_out/ncu_v${V}.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_v${V}.log
