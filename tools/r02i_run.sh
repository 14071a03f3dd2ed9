mkdir -p gpurun_out/r02i
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02i/pytest.log 2>&1
timeout 600 python tools/ab_exp.py C 0,4 > gpurun_out/r02i/ab.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_composite_staged|k_emit_rows|k_emit_big|k_count_big|k_ranges|k_radix_hist|k_scan" -c 9 -o gpurun_out/r02i/full2 python tools/prof_frame.py C 1 > gpurun_out/r02i/full2.log 2>&1
echo done
