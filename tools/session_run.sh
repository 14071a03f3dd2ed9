O=gpurun_out/s3ag; mkdir -p $O
timeout 600 python tools/exp_equal.py P4K 0 4096 > $O/equal.txt 2>&1
timeout 600 python tools/ab_exp.py P4K 0,4096 > $O/abP4K.txt 2>&1
echo done
