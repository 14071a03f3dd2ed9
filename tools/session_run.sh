O=gpurun_out/s3aa; mkdir -p $O
timeout 600 python tools/ab_time.py C 10 2 > $O/abC2.txt 2>&1
CR_EXP=4096 timeout 600 python tools/ab_time.py C 10 2 >> $O/abC2.txt 2>&1
timeout 600 python tools/exp_equal.py A 0 4096 2 > $O/equal.txt 2>&1
bash tools/refresh_r02c.sh
bash tools/refresh_r02b.sh
echo done
