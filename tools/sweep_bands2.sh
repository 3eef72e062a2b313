# column bands in the length-class order (cfg3) + regression check of the band configs
source tools/sweep_layout.sh --defs-only
run b2_cfg3_auto --config cfg3
run b2_cfg3_K4 --config cfg3 --column-bands 4
run b2_cfg3_off --config cfg3 --column-bands 1
run b2_cfg3s_K2 --config cfg3s --column-bands 2
run b2_cfg5s_auto --config cfg5s
run b2_cfg4_auto --config cfg4 --permutation none
run b2_cfg2_auto --config cfg2
for t in b2_cfg3_auto b2_cfg3_K4 b2_cfg4_auto b2_cfg5s_auto; do
  python -c "import json; d=json.loads(open('gpurun_out/sweep/$t.log').read().strip().splitlines()[-1]); c=d['config']['layout_choices']; print('$t', c.get('order'), c.get('column_bands'), c.get('light_row_max'))"
done
