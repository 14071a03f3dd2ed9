mkdir -p gpurun_out/r02c
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_composite_staged -c 1 -o gpurun_out/r02c/comp python tools/prof_frame.py C 1 > gpurun_out/r02c/ncu_comp.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_countv -c 1 -o gpurun_out/r02c/count python tools/prof_frame.py C 1 > gpurun_out/r02c/ncu_count.log 2>&1
echo done
