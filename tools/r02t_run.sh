mkdir -p gpurun_out/r02t
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02t/pytest.log 2>&1
timeout 300 python tools/ab_time.py C 15 > gpurun_out/r02t/abC.txt 2>&1
timeout 300 python tools/ab_exp.py C 0 69:74 > gpurun_out/r02t/ab_band.txt 2>&1
for R in 2 4 8; do timeout 900 python tools/band_cost.py C $R refined > gpurun_out/r02t/band_costs_R${R}_refined.txt 2>&1; done
echo done
