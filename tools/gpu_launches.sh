# per-kernel launch list (ncu, one pass) for a bench config: tools/gpu_launches.sh CFG [extra bench args]
mkdir -p gpurun_out
CFG=$1; shift
timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum --clock-control none -k "regex:(sell32|sell32_pipe|heavy_chunk|long_row)_kernel" -s ${SKIP:-30} -c ${COUNT:-12} --csv --log-file gpurun_out/launch_$CFG.csv python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-spmv --no-extra "$@" > /dev/null 2>&1; echo "ncu rc=$?"
