#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python scripts/overlap_bench.py --sim 8 --bwd-ms 1.0 > $O/overlap_sim8.json 2> $O/overlap_sim8.err
timeout 600 python scripts/overlap_bench.py --sim 8 --bwd-ms 2.0 --dtype fp16 > $O/overlap_sim8_fp16.json 2> $O/overlap_sim8_fp16.err
timeout 600 python scripts/sweep.py --sim 8 --max-mb 256 --algos oneshot,twoshot,auto,nccl > $O/sweep_sim8.jsonl 2> $O/sweep_sim8.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
    bench.py --gpus 2 --steps 10 --warmup 3 --min-warmup-s 0 > $O/bench_n2_1gpu.json 2> $O/bench_n2_1gpu.err
echo "torchrun rc=$?" >> $O/bench_n2_1gpu.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
echo ALL DONE
