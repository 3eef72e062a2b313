# default (autotuned) layout on the structured configs; compare with tools/sweep_layout.sh
source tools/sweep_layout.sh --defs-only
run auto_cfg4s_none --config cfg4s --permutation none
run auto_cfg4s --config cfg4s
run auto_cfg3s --config cfg3s
run auto_cfg4_none --config cfg4 --permutation none
run auto_cfg3 --config cfg3
run auto_cfg2 --config cfg2
for t in auto_cfg4s_none auto_cfg4s auto_cfg3s auto_cfg4_none auto_cfg3 auto_cfg2; do
  python -c "import json,sys; d=json.loads(open('gpurun_out/sweep/$t.log').read().strip().splitlines()[-1]); print('$t', d['config']['layout_choices'].get('order'), d['config']['layout_choices'].get('order_spans'), sorted(set(d['config']['layout_choices']['light_row_max'].items()))[:6])"
  grep -o "setup [0-9.]*s" gpurun_out/sweep/$t.log | head -1
done
