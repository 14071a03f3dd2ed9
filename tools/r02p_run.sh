mkdir -p gpurun_out/r02p
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02p/pytest.log 2>&1
timeout 300 python tools/ab_time.py C 15 > gpurun_out/r02p/abC.txt 2>&1
for R in 2 4 8; do timeout 600 python tools/band_cost.py C $R refined > gpurun_out/r02p/band_costs_R${R}_refined.txt 2>&1; done
timeout 600 python bench.py > gpurun_out/r02p/bench.log 2>&1
echo done
