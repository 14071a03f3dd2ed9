mkdir -p gpurun_out/r02g
timeout 600 python tools/ab_exp.py C 0,1,2,3 > gpurun_out/r02g/ab_full.txt 2>&1
timeout 600 python tools/ab_exp.py C 0,1,2,3 69:74 > gpurun_out/r02g/ab_band.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02g/launch_band.csv python tools/prof_frame.py C 2 8 0 1 69:74 > /dev/null 2>&1
CR_EXP=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02g/launch_band_exp2.csv python tools/prof_frame.py C 2 8 0 1 69:74 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02g/launch_full.csv python tools/prof_frame.py C 2 > /dev/null 2>&1
echo done
