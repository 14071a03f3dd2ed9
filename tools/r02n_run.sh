mkdir -p gpurun_out/r02n
timeout 300 python tools/rb_diff.py A > gpurun_out/r02n/diffA.txt 2>&1
timeout 300 python tools/rb_diff.py C > gpurun_out/r02n/diffC.txt 2>&1
timeout 600 python tools/ab_exp.py C 0,8 > gpurun_out/r02n/ab.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_rowbin|k_rowscan|k_colsort" -c 3 -o gpurun_out/r02n/rb python tools/prof_frame.py C 1 > gpurun_out/r02n/rb.log 2>&1
CR_EXP=8 timeout 600 ncu --set full --clock-control none -k regex:"k_radix_onesweep|k_emit_rows" -c 7 -o gpurun_out/r02n/lsd python tools/prof_frame.py C 1 > gpurun_out/r02n/lsd.log 2>&1
echo done
