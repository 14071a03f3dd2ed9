#!/bin/bash
# usage (under gpurun): bash tools/refresh_profiles.sh OUTDIR
# Round profile refresh: bench lines of every config, per-kernel ncu table and
# launch list of config C, full ncu capture of the composite, band costs.
O=${1:-gpurun_out/prof}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > $O/gpu.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_configC.json 2> $O/bench_configC.err
for C in A B D E P2K P4K; do
  timeout 900 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_config$C.json 2> $O/bench_config$C.err
done
bash tools/prof_all.sh r01 C > /dev/null 2>&1
cp gpurun_out/ncu_table_r01.txt $O/ncu_kernels_configC.txt
cp gpurun_out/launches_r01.csv $O/launches_configC.csv
python tools/launches.py $O/launches_configC.csv > $O/launches_configC.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_composite_staged" -c 1 -o $O/composite_full python tools/prof_frame.py C 1 > /dev/null 2>&1
python tools/ncu_details.py $O/composite_full.ncu-rep > $O/composite_full_summary.txt 2>&1
for R in 2 4 8; do python tools/band_cost.py C $R refined > $O/band_costs_R${R}_refined.txt 2>&1; done
echo done
