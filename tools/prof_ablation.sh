#!/bin/bash
# usage (under gpurun): bash tools/prof_ablation.sh TAG [config]
# ncu counters of the composite: B200 staged kernel vs the paper's thread-per-subpixel
# kernel with and without View-coherent Remapping (one launch each)
TAG=$1; CFG=${2:-C}
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__thread_inst_executed_per_inst_executed.ratio,sm__inst_executed.avg.per_cycle_active,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,smsp__inst_executed.sum
for K in "0 1" "1 1" "1 0"; do
  set -- $K
  ncu --metrics $M --clock-control none -k regex:k_composite -c 1 --csv python tools/prof_frame.py $CFG 1 8 $1 $2 > gpurun_out/abl_${TAG}_k$1_r$2.csv 2>/dev/null
done
echo done
