mkdir -p gpurun_out/r02d
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02d/pytest.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02d/bench.log 2>&1
timeout 900 python -m paper_2605_04509_b200.quality C 2,4,8,10,16 > gpurun_out/r02d/quality_C.md 2>&1
echo done
