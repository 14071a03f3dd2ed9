O=gpurun_out/s3af; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
timeout 600 python tools/ab_time.py C 15 > $O/abC.txt 2>&1
echo done
