# first-touch column order inside the length classes vs plain class order
source tools/sweep_layout.sh --defs-only
run t_cfg2_on --config cfg2
run t_cfg2_off --config cfg2 --no-first-touch
run t_cfg3s_on --config cfg3s
run t_cfg3s_off --config cfg3s --no-first-touch
run t_cfg3_on --config cfg3
run t_cfg3_off --config cfg3 --no-first-touch
run t_cfg4s_on --config cfg4s
