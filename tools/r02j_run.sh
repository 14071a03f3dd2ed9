mkdir -p gpurun_out/r02j
for cfg in A B C; do CR_DEBUG=0 timeout 300 python tools/rb_check.py $cfg >> gpurun_out/r02j/rb_check.txt 2>&1; done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02j/pytest.log 2>&1
timeout 600 python tools/ab_exp.py C 0,8 > gpurun_out/r02j/ab.txt 2>&1
echo done
