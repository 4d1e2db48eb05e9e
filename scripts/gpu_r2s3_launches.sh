#!/bin/bash
# Round 2, session 3: the launch list of the benched command (ncu
# gpu__time_duration, cold / serialised), after the same command ran clean.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > $O/r2s3_launches_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/r2s3_launches.csv $CMD > $O/r2s3_launches_ncu.log 2>&1; echo "ncu rc=$?"
python scripts/ncu_summary.py launches $O/r2s3_launches.csv > $O/r2s3_launches_summary.json; cat $O/r2s3_launches_summary.json | head -30
