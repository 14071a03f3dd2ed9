#!/bin/bash
# Round-2 final refresh (session 3), part 1 (under gpurun): GPU tests, smoke,
# bench lines of every config, the reference arm, ablation, a 2-rank gloo run.
O=gpurun_out/r02final; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total,driver_version --format=csv > $O/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_configC.json 2> $O/bench_configC.err
for C in A B D E P2K P4K; do
  timeout 900 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_config$C.json 2> $O/bench_config$C.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 python bench.py --steps 5 --warmup 3 --ablation --no-cpu-baseline --no-fullframe --no-traffic > /dev/null 2> $O/ablation_configC.err
grep '\[ablation\]' $O/ablation_configC.err > $O/ablation_configC.txt
CR_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 5 --warmup 3 > $O/bench_gloo2.json 2> $O/bench_gloo2.err
echo done
