mkdir -p gpurun_out/r02a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02a/pytest.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_run.py all > gpurun_out/r02a/memcheck.log 2>&1
timeout 900 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_run.py A > gpurun_out/r02a/racecheck_A.log 2>&1
CR_SAN_M=50000 timeout 900 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_run.py B > gpurun_out/r02a/racecheck_B.log 2>&1
timeout 900 compute-sanitizer --tool synccheck --print-limit 50 python tools/sanitize_run.py A > gpurun_out/r02a/synccheck_A.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-fullframe > gpurun_out/r02a/bench.log 2>&1
echo done
