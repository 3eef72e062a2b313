# ncu --set full of cfg4's (MCF, +-1 values, UNIT codec) two main-loop kernels
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:sell32_pipe_kernel<.*Op(Primal|Dual)' -s 6 -c 2 -o gpurun_out/prof_cfg4 python bench.py --config cfg4 --permutation none --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-spmv --no-extra > gpurun_out/ncu_cfg4.log 2>&1; echo "ncu cfg4 rc=$?"
python tools/ncu_summary.py gpurun_out/prof_cfg4.ncu-rep gpurun_out/ncu_cfg4.md 2>&1 | tail -2
