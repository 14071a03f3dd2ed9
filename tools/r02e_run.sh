mkdir -p gpurun_out/r02e
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "config_d or config_e or paper_display or config_c" --durations=10 > gpurun_out/r02e/pytest_big.log 2>&1
timeout 2400 python tools/oracle_timing.py A,A1,B,C > gpurun_out/r02e/oracle_timings.md 2>&1
echo done
