O=gpurun_out/s3k; mkdir -p $O
./tools/x2check/vrc_check > $O/vrc.txt 2>&1
timeout 600 python tools/dbg_counts.py > $O/dbg_cur.txt 2>&1
timeout 600 python tools/exp_equal.py C 0 2624 > $O/equal.txt 2>&1
timeout 600 python tools/ab_exp.py C 0,2624 > $O/abC.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1
echo done
