#!/bin/bash
# Round-2 evidence refresh: launch list of the bench command (ncu
# gpu__time_duration, cold + serialised: compare shares), ncu --set full of
# the bench's kernel (fp32, fp16) -> profiles/ncu summaries and traffic.json.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 5 --warmup 3 --min-warmup-s 0 --no-cpu-baseline --no-e2e > $O/bench_ncu.log 2>&1
for dt in fp32 fp16; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_update_direct -s 3 -c 1 \
    -o $O/prof_update_direct_$dt -f python bench.py --steps 3 --warmup 3 --min-warmup-s 0 --no-cpu-baseline --no-e2e --dtype $dt > $O/prof_$dt.log 2>&1
done
echo ALL DONE
