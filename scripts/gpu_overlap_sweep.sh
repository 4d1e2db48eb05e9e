#!/bin/bash
# BASELINE config 4 sweep (bucket size x dtype) with the calibrated,
# interleaved-median overlap_bench: N = 1 real communicator, 8 simulated ranks.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
rm -f $O/overlap_sweep.jsonl
for dt in fp32 fp16; do for mb in 4 8 16 25; do
  timeout 600 python scripts/overlap_bench.py --bwd-ms 1.0 --bucket-mb $mb --dtype $dt >> $O/overlap_sweep.jsonl 2>> $O/overlap_sweep.err
done; done
for mb in 4 8 16 25; do
  timeout 600 python scripts/overlap_bench.py --sim 8 --bwd-ms 4.0 --bucket-mb $mb >> $O/overlap_sweep.jsonl 2>> $O/overlap_sweep.err
done
echo ALL DONE
