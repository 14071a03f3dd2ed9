#!/bin/bash
# usage (under gpurun): bash tools/prof_kernels.sh TAG "regex1|regex2" [config]
TAG=$1; RE=$2; CFG=${3:-C}
ncu --set full --clock-control none --import-source on -k regex:"$RE" -c 1 -o gpurun_out/prof_$TAG python tools/prof_frame.py $CFG 1 > gpurun_out/prof_$TAG.log 2>&1
echo done
