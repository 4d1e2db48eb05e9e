#!/bin/bash
# Refresh: ncu --set full of k_pack (fp32, fp16), k_update_sgd, k_update_direct, and the bench launch list.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for k in k_pack k_update_sgd; do
  for dt in fp32 fp16; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o $O/prof_${k}_$dt -f python scripts/prof_driver.py --mode n1 --dtype $dt > $O/prof_${k}_$dt.log 2>&1
  done
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 5 --warmup 3 --min-warmup-s 0 --no-cpu-baseline --no-e2e > $O/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_update_direct -s 3 -c 1 \
    -o $O/prof_update_direct -f python bench.py --steps 3 --warmup 3 --min-warmup-s 0 --no-cpu-baseline --no-e2e > $O/prof.log 2>&1
echo ALL DONE
