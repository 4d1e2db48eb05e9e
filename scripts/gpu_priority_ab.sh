#!/bin/bash
# Config-4 A/B: communication-stream priority (high vs low relative to the
# backward) x grid cap x bucket size, graph and eager launch; plus the
# robustness-seed parity tests.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "robustness" > $O/pytest_seeds.log 2>&1; echo "rc=$?" >> $O/pytest_seeds.log
rm -f $O/overlap_prio.jsonl
for launch in graph eager; do
  for mb in 4 16 25; do
    for sc in 0 64; do
      for pr in high low; do
        timeout 300 python scripts/overlap_bench.py --bwd-ms 1.0 --bucket-mb $mb --stream-ctas $sc \
          --comm-priority $pr --launch $launch --reps 9 >> $O/overlap_prio.jsonl 2>> $O/overlap_prio.err
      done
    done
  done
done
echo ALL DONE
