O=gpurun_out/s3q; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_composite_pairs" -c 1 -o $O/comp python tools/prof_frame.py C 1 > $O/ncu.log 2>&1
echo done
