#!/bin/bash
# usage (under gpurun): bash tools/prof_all.sh TAG [config]
# per-kernel DRAM bytes / duration / IPC / occupancy of one frame (frame 2), summarised on the box
TAG=$1; CFG=${2:-C}
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.avg.per_cycle_active,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum
ncu --metrics $M --clock-control none -c 70 -o /tmp/full_$TAG python tools/prof_frame.py $CFG 1 > gpurun_out/full_$TAG.log 2>&1
python tools/ncu_table.py /tmp/full_$TAG.ncu-rep > gpurun_out/ncu_table_$TAG.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python tools/prof_frame.py $CFG 2 > /dev/null 2>&1
echo done
