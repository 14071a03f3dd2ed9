mkdir -p gpurun_out/r02b
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02b/pytest.log 2>&1
for cfg in C B; do timeout 300 python tools/ab_time.py $cfg 15 >> gpurun_out/r02b/time.log 2>&1; done
echo done
