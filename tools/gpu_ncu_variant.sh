# ncu --set full of one product kernel per variant: VARIANTS (default "1"), CFG (cfg2), KREGEX
mkdir -p gpurun_out
CFG=${CFG:-cfg2}
for v in ${VARIANTS:-1}; do
  if [ "$v" = 0 ]; then K=${KREGEX:-'regex:sell32_kernel<.*OpDual'}; else K=${KREGEX:-'regex:sell_tma_kernel<.*OpDual'}; fi
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$K" -s 20 -c 1 \
    -o gpurun_out/prof_${CFG}_v$v python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-spmv --no-extra \
    --tuning sell_variant=$v > gpurun_out/ncu_${CFG}_v$v.log 2>&1; echo "ncu v$v rc=$?"
  python tools/ncu_summary.py gpurun_out/prof_${CFG}_v$v.ncu-rep gpurun_out/ncu_${CFG}_v$v.md 2>&1 | tail -2
done
