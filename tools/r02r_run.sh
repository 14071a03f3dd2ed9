mkdir -p gpurun_out/r02r
for cfg in A B C; do timeout 600 python tools/exp_equal.py $cfg 0 4 >> gpurun_out/r02r/equal.txt 2>&1; done
timeout 600 python tools/ab_exp.py C 0,4 > gpurun_out/r02r/ab.txt 2>&1
timeout 300 python tools/ab_exp.py B 0,4 > gpurun_out/r02r/abB.txt 2>&1
echo done
