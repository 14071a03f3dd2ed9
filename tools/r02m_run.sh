mkdir -p gpurun_out/r02m
timeout 300 python tools/rb_diff.py A > gpurun_out/r02m/diffA.txt 2>&1
timeout 300 python tools/rb_diff.py C > gpurun_out/r02m/diffC.txt 2>&1
timeout 600 python tools/ab_exp.py C 0,8 > gpurun_out/r02m/ab.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_rowbin|k_rowscan|k_colsort|k_tile_bases|k_ranges_rb|k_count_big_rb" -c 6 -o gpurun_out/r02m/rb python tools/prof_frame.py C 1 > gpurun_out/r02m/rb.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02m/pytest.log 2>&1
echo done
