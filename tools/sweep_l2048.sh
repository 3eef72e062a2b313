# cfg4 coupling rows (1300 entries) in SELL lanes: light_row_max 2048 in the layout order
source tools/sweep_layout.sh --defs-only
run l_cfg4_nat_L256 --config cfg4 --permutation none --natural-order --light-row-max 256 --column-bands 1
run l_cfg4_nat_L2048 --config cfg4 --permutation none --natural-order --light-row-max 2048 --column-bands 1
run l_cfg4_nat_L2048_b16 --config cfg4 --permutation none --natural-order --light-row-max 2048 --column-bands 16
run l_cfg4s_nat_L256 --config cfg4s --permutation none --natural-order --light-row-max 256
run l_cfg3_L1024 --config cfg3 --light-row-max 1024
