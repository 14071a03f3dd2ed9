O=gpurun_out/s3r; mkdir -p $O
timeout 600 python tools/exp_equal.py C 0 64 > $O/equal.txt 2>&1
bash tools/ab_lib.sh build/lib9.so C $O/ab9.txt
timeout 600 python tools/ab_exp.py B 0 > $O/abB.txt 2>&1
CR_LIB=build/lib9.so timeout 600 python tools/ab_exp.py B 0 >> $O/abB.txt 2>&1
echo done
