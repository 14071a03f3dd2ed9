#!/bin/bash
# usage (under gpurun): bash tools/prof_all.sh TAG [config]  -- full ncu capture of every kernel of one frame
TAG=$1; CFG=${2:-C}
ncu --set full --clock-control none --import-source on -s 60 -c 60 -o gpurun_out/full_$TAG python tools/prof_frame.py $CFG 2 > gpurun_out/full_$TAG.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python tools/prof_frame.py $CFG 2 > /dev/null 2>&1
echo done
