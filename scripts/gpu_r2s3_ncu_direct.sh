#!/bin/bash
# Round 2, session 3: ncu --set full of the bench's kernel (k_update_direct,
# fp32) on the final build, after the same command ran clean.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
CMD="python bench.py --steps 3 --warmup 3 --min-warmup-s 0 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > $O/r2s3_direct_plain.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_update_direct -s 5 -c 1 \
  -o $O/r2s3_k_update_direct $CMD > $O/r2s3_ncu_direct.log 2>&1; echo "ncu rc=$?"
tail -3 $O/r2s3_ncu_direct.log
