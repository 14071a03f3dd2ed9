O=gpurun_out/s3z; mkdir -p $O
timeout 600 python tools/exp_equal.py P2K 0 4096 > $O/equal.txt 2>&1
timeout 600 python tools/exp_equal.py A 0 4096 4 >> $O/equal.txt 2>&1
timeout 600 python tools/ab_exp.py P2K 0,4096 > $O/abP2K.txt 2>&1
timeout 600 python tools/ab_time.py C 15 4 > $O/abC4.txt 2>&1
CR_EXP=4096 timeout 600 python tools/ab_time.py C 15 4 >> $O/abC4.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1
echo done
