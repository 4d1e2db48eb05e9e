#!/bin/bash
# Round-end validation: scripts/gpu_check.sh (smoke, pytest -m gpu, bench fp32/fp16,
# launch list, ncu --set full of the bench kernel), the reference arm, and the
# oracle timed on the box's host cores, single-threaded and partitioned (SURVEY d.5).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
bash scripts/gpu_check.sh
O=gpurun_out
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
rm -f $O/oracle_times.jsonl
for dt in fp32 fp16; do for n in 1 2 4 8; do
  timeout 600 python -m oracle --config r50 --workers $n --dtype $dt --steps 3 --time --threads 0 >> $O/oracle_times.jsonl 2>> $O/oracle_times.err
done; done
echo FINAL DONE
