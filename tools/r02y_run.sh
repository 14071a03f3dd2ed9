mkdir -p gpurun_out/r02y
for cfg in A C B P4K; do timeout 600 python tools/exp_equal.py $cfg 0 4 >> gpurun_out/r02y/equal.txt 2>&1; done
timeout 600 python tools/ab_exp.py C 0,4 > gpurun_out/r02y/ab.txt 2>&1
timeout 300 python tools/ab_exp.py P4K 0,4 > gpurun_out/r02y/abP4K.txt 2>&1
timeout 300 python tools/ab_exp.py B 0,4 > gpurun_out/r02y/abB.txt 2>&1
echo done
