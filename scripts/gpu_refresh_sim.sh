#!/bin/bash
# Refresh the simulated-N / time-sliced evidence for the current build:
# kernel bench (whole-step schedules, N = 2/4/8 simulated), config-5 sweep and
# config-4 overlap mechanics, and bench.py under torchrun with 8 ranks on the one GPU.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python scripts/kernel_bench.py --worlds 2,4,8 > $O/kernel_bench_sim.jsonl 2> $O/kernel_bench_sim.err
timeout 900 python scripts/sweep.py --sim 8 --max-mb 1024 --algos oneshot,twoshot,auto > $O/sweep_sim8.jsonl 2> $O/sweep_sim8.err
timeout 600 python scripts/overlap_bench.py --bwd-ms 1.0 > $O/overlap_n1.json 2> $O/overlap_n1.err
timeout 600 python scripts/overlap_bench.py --sim 8 --bwd-ms 1.0 > $O/overlap_sim8.json 2> $O/overlap_sim8.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29513 \
    bench.py --gpus 8 --steps 10 --warmup 3 --min-warmup-s 0 > $O/bench_n8_1gpu.json 2> $O/bench_n8_1gpu.err
echo "torchrun rc=$?" >> $O/bench_n8_1gpu.err
echo ALL DONE
