mkdir -p gpurun_out/r02s
for cfg in A C; do timeout 600 python tools/exp_equal.py $cfg 0 4 >> gpurun_out/r02s/equal.txt 2>&1; done
timeout 600 python tools/ab_exp.py C 0,4 > gpurun_out/r02s/ab.txt 2>&1
timeout 300 python tools/ab_exp.py P4K 0,4 > gpurun_out/r02s/abP4K.txt 2>&1
echo done
