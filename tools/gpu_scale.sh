# Strong-scaling lines on a multi-GPU box (never run in this project: one GPU
# per call here). For each N in NS (default "1 2 4 8") and each config in
# CFGS (default "cfg2 cfg3"): torchrun one rank per GPU, the NCCL executor
# (sharded ordered exchanges, CUDA graphs); COMM=peer for the in-kernel
# peer-memory exchange. Lines land in gpurun_out/scale_<cfg>_n<N>.log.
mkdir -p gpurun_out
for cfg in ${CFGS:-cfg2 cfg3}; do
  E2E=""; [ "$cfg" != cfg2 ] && E2E="--no-e2e"      # time to tolerance only on the metric's config
  for n in ${NS:-1 2 4 8}; do
    if [ "$n" = 1 ]; then
      timeout 1200 python bench.py --config $cfg --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-spmv --no-extra $E2E \
        > gpurun_out/scale_${cfg}_n$n.log 2>&1
    else
      timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port $((29600 + n)) bench.py --gpus $n --config $cfg --steps ${STEPS:-10} --warmup 3 \
        --comm ${COMM:-nccl} --no-cpu-baseline $E2E > gpurun_out/scale_${cfg}_n$n.log 2>&1
    fi
    python - "gpurun_out/scale_${cfg}_n$n.log" "$cfg n=$n" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], "it/s", round(d["value"], 1), "us/iter", round(d["roofline"]["seconds_per_launch"] * 1e6, 1),
          "grid", d["config"].get("grid"), "e2e", (d.get("e2e") or {}).get("time_to_tol_s"))
except Exception as e:
    print(sys.argv[2], "parse failed", e); print(open(sys.argv[1]).read()[-1500:])
PY
  done
done
