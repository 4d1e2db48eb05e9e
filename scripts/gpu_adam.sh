#!/bin/bash
# NEXT-1 measurement: kernel bench (N = 1, incl. Adam) + ncu --set full of k_update_adam.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || echo "BUILD FAILED" >> $O/build.log
timeout 600 python scripts/kernel_bench.py --worlds 1 > $O/kernel_bench_n1.jsonl 2> $O/kernel_bench_n1.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_update_adam -s 2 -c 1 \
    -o $O/prof_k_update_adam -f python scripts/prof_driver.py --mode adam > $O/prof_adam.log 2>&1
echo ALL DONE
