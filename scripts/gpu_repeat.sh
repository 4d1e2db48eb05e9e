#!/bin/bash
# Run-to-run spread of the headline bench: five back-to-back `python bench.py` runs
# (fp32), then three fp16, on one box.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
rm -f $O/bench_repeat.jsonl
for r in 1 2 3 4 5; do timeout 600 python bench.py --no-cpu-baseline >> $O/bench_repeat.jsonl 2>> $O/bench_repeat.err; done
for r in 1 2 3; do timeout 600 python bench.py --dtype fp16 --no-cpu-baseline >> $O/bench_repeat.jsonl 2>> $O/bench_repeat.err; done
echo ALL DONE
