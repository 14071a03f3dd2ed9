O=gpurun_out/s3ab; mkdir -p $O
timeout 600 python tools/exp_equal.py C 0 4096 > $O/equal.txt 2>&1
timeout 900 python tools/ab_exp.py C 0,4096 > $O/abC.txt 2>&1
timeout 600 python tools/ab_exp.py B 0,4096 > $O/abB.txt 2>&1
echo done
