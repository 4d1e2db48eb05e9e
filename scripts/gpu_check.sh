#!/bin/bash
# One gpurun call: smoke, GPU tests, bench, launch list, one ncu --set full capture.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
nvidia-smi > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || echo "BUILD FAILED" >> $O/build.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --dtype fp16 --no-cpu-baseline > $O/bench_fp16.json 2> $O/bench_fp16.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 5 --warmup 3 --min-warmup-s 0 --no-cpu-baseline --no-e2e > $O/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_update_direct -s 3 -c 1 \
    -o $O/prof_update_direct -f python bench.py --steps 3 --warmup 3 --min-warmup-s 0 --no-cpu-baseline --no-e2e > $O/prof.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_update_direct -s 3 -c 1 \
    -o $O/prof_update_direct_fp16 -f python bench.py --dtype fp16 --steps 3 --warmup 3 --min-warmup-s 0 --no-cpu-baseline --no-e2e > $O/prof16.log 2>&1
echo ALL DONE
