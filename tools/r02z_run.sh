mkdir -p gpurun_out/r02z
timeout 300 python tools/exp_equal.py C 0 16 > gpurun_out/r02z/equal.txt 2>&1
timeout 600 python tools/ab_exp.py C 0,16 > gpurun_out/r02z/ab.txt 2>&1
bash tools/ab_lib.sh tools/prev/libprev.so C gpurun_out/r02z/ab_lib.txt
echo done
