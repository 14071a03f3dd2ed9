O=gpurun_out/s3p; mkdir -p $O
timeout 600 python tools/exp_equal.py C 0 64 > $O/equal.txt 2>&1
timeout 600 python tools/exp_equal.py P4K 0 64 >> $O/equal.txt 2>&1
timeout 900 python tools/ab_exp.py C 0 > $O/abC.txt 2>&1
timeout 600 python tools/ab_exp.py B 0 > $O/abB.txt 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_run.py all > $O/memcheck.log 2>&1
timeout 900 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_run.py A > $O/racecheck_A.log 2>&1
echo done
