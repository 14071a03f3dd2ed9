# round-2 (session 2) baseline captures: full ncu of count, composite, preprocess, emission; launch list
mkdir -p gpurun_out/r02h
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_countv|k_composite_staged|k_preprocess|k_emit_rows|k_radix_onesweep" -c 6 -o gpurun_out/r02h/full python tools/prof_frame.py C 1 > gpurun_out/r02h/full.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02h/launch_full.csv python tools/prof_frame.py C 2 > /dev/null 2>&1
echo done
