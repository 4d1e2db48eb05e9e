#!/bin/bash
# Simulated-N evidence on one GPU: kernel bench incl. whole-step schedules,
# config-5 sweep mechanics, config-4 overlap, ncu of the fused/sharded kernels.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python scripts/kernel_bench.py --worlds 2,4,8 > $O/kernel_bench_sim.jsonl 2> $O/kernel_bench_sim.err
timeout 900 python scripts/sweep.py --sim 8 --max-mb 1024 --algos oneshot,twoshot,auto > $O/sweep_sim8.jsonl 2> $O/sweep_sim8.err
timeout 600 python scripts/overlap_bench.py --bwd-ms 1.0 > $O/overlap_n1.json 2> $O/overlap_n1.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_update_gather -s 1 -c 1 \
    -o $O/prof_k_update_gather_sim8 -f python scripts/prof_driver.py --mode fused8 > $O/prof_fused.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_update_chunk|k_gather_params" -s 8 -c 2 \
    -o $O/prof_sharded_sim8 -f python scripts/prof_driver.py --mode sharded8 > $O/prof_sharded.log 2>&1
echo ALL DONE
