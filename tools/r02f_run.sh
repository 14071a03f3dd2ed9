mkdir -p gpurun_out/r02f
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "not config_d and not config_e and not paper_display" > gpurun_out/r02f/pytest.log 2>&1
for cfg in C B; do timeout 300 python tools/ab_time.py $cfg 15 >> gpurun_out/r02f/time.log 2>&1; done
timeout 600 python tools/band_cost.py C 8 refined > gpurun_out/r02f/band_R8.txt 2>&1
timeout 600 python tools/band_cost.py C 4 refined > gpurun_out/r02f/band_R4.txt 2>&1
echo done
