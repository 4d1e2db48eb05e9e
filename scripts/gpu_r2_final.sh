#!/bin/bash
# Round-2 final validation on a fresh box: build + smoke, the whole GPU
# suite, the driver's bench command (N = 1, 20 steps after 5) and the
# contract default (100 after 20), fp16, and the reference arm.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/final_smoke.log 2>&1 || echo "BUILD/SMOKE FAILED" >> $O/final_smoke.log
timeout 2700 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider --durations=15 > $O/final_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/final_pytest_gpu.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/final_bench_driver_cmd.json 2> $O/final_bench_driver_cmd.err
timeout 600 python bench.py > $O/final_bench_fp32.json 2> $O/final_bench_fp32.err
timeout 600 python bench.py --dtype fp16 > $O/final_bench_fp16.json 2> $O/final_bench_fp16.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/final_bench_reference.json 2> $O/final_bench_reference.err
echo ALL DONE
