#!/bin/bash
# Round 2, session 3: the emulated tests incl. the slow-rank mid-barrier test
# and its negative control; the emulated config-5 sweep with graph replay.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; tail -30 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_emulated.py -m gpu -q -p no:cacheprovider -rA --durations=8 > $O/r2s3_emulated2.txt 2>&1; echo "emulated rc=$?" >> $O/r2s3_emulated2.txt
tail -4 $O/r2s3_emulated2.txt
timeout 900 python scripts/emulated_bench.py --sweep --worlds 2,4,8 > $O/r2s3_emulated_sweep.jsonl 2> $O/r2s3_emulated_sweep.err; echo "sweep rc=$?"
cat $O/r2s3_emulated_sweep.jsonl
