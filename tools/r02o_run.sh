mkdir -p gpurun_out/r02o
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02o/pytest.log 2>&1
timeout 300 python tools/ab_exp.py C 0,32 > gpurun_out/r02o/ab.txt 2>&1
for R in 2 4 8; do timeout 600 python tools/band_cost.py C $R refined > gpurun_out/r02o/band_costs_R${R}_refined.txt 2>&1; done
echo done
