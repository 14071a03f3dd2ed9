#!/bin/bash
# Round-2 refresh, part 2 (under gpurun): ncu per-kernel table + launch list
# of config C, full captures of the composite and the count, band costs,
O=gpurun_out/r02final; mkdir -p $O
bash tools/prof_all.sh r02 C > /dev/null 2>&1
cp gpurun_out/ncu_table_r02.txt $O/ncu_kernels_configC.txt
cp gpurun_out/launches_r02.csv $O/launches_configC.csv
python tools/launches.py $O/launches_configC.csv > $O/launches_configC.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_composite_pairs|k_countv" -c 2 -o $O/comp_count_full python tools/prof_frame.py C 1 > /dev/null 2>&1
python tools/ncu_details.py $O/comp_count_full.ncu-rep > $O/comp_count_full_summary.txt 2>&1
python tools/ncu_lines.py $O/comp_count_full.ncu-rep k_composite 40 > $O/composite_lines.txt 2>&1
python tools/ncu_lines.py $O/comp_count_full.ncu-rep k_countv 40 > $O/count_lines.txt 2>&1
for R in 2 4 8; do timeout 900 python tools/band_cost.py C $R refined > $O/band_costs_R${R}_refined.txt 2>&1; done
echo done
