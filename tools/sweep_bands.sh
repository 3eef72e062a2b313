# column bands (BandedCsr) on the configs whose gather vectors exceed L2
source tools/sweep_layout.sh --defs-only
run bands_cfg5s_auto --config cfg5s
run bands_cfg5s_off --config cfg5s --column-bands 1
run bands_cfg5s_K8 --config cfg5s --column-bands 8
run bands_cfg3_auto --config cfg3
run bands_cfg3_off --config cfg3 --column-bands 1
run bands_cfg4_auto --config cfg4 --permutation none
run bands_cfg2_auto --config cfg2
for t in bands_cfg5s_auto bands_cfg3_auto bands_cfg4_auto bands_cfg5s_K8; do
  python -c "import json; d=json.loads(open('gpurun_out/sweep/$t.log').read().strip().splitlines()[-1]); c=d['config']['layout_choices']; print('$t', c.get('order'), c.get('column_bands'), c.get('light_row_max'))"
done
