O=gpurun_out/s3s; mkdir -p $O
./tools/x2check/vrc_check > $O/vrc.txt 2>&1
bash tools/ab_lib.sh build/libhead.so C $O/ab_sqrt.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x > $O/pytest.log 2>&1
bash tools/refresh_r02b.sh
echo done
