# column bands with evict-first carries: band sizes on cfg3 / cfg5s / cfg4
source tools/sweep_layout.sh --defs-only
run b3_cfg3_off --config cfg3 --column-bands 1
run b3_cfg3_K4 --config cfg3 --column-bands 4
run b3_cfg3_K8 --config cfg3 --column-bands 8
run b3_cfg3_auto24 --config cfg3 --band-mb 24
run b3_cfg5s_auto --config cfg5s
run b3_cfg5s_auto24 --config cfg5s --band-mb 24
run b3_cfg5s_auto96 --config cfg5s --band-mb 96
run b3_cfg4_auto --config cfg4 --permutation none
run b3_cfg4_auto24 --config cfg4 --permutation none --band-mb 24
for t in b3_cfg3_auto24 b3_cfg5s_auto b3_cfg5s_auto24 b3_cfg5s_auto96 b3_cfg4_auto b3_cfg4_auto24; do
  python -c "import json; d=json.loads(open('gpurun_out/sweep/$t.log').read().strip().splitlines()[-1]); c=d['config']['layout_choices']; print('$t', c.get('order'), c.get('column_bands'))"
done
