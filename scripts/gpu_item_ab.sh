#!/bin/bash
# A/B of the L2 evict_last policy on work-item descriptor loads (build switch).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
rm -f $O/item_ab.jsonl
for rep in 1 2 3; do for mode in plain evict_last; do
  if [ $mode = evict_last ]; then export CMN_EXTRA_NVFLAGS=-DCMN_ITEM_EVICT_LAST; else unset CMN_EXTRA_NVFLAGS; fi
  python -c "from paper_1908_00213_b200 import build; build.build(force=True)" > $O/build_$mode.log 2>&1
  timeout 300 python bench.py --steps 200 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json, sys
d = json.loads(sys.stdin.read()); print(json.dumps({'mode': '$mode', 'rep': $rep, 'bench_us': d['value']}))" >> $O/item_ab.jsonl
  timeout 300 python scripts/kernel_bench.py --worlds 1 2>/dev/null | python -c "
import json, sys
for l in sys.stdin:
    d = json.loads(l); print(json.dumps({'mode': '$mode', 'rep': $rep, 'dtype': d['dtype'], 'pack_us': d['allreduce_incl_pack_us']}))" >> $O/item_ab.jsonl
done; done
unset CMN_EXTRA_NVFLAGS
python -c "from paper_1908_00213_b200 import build; build.build(force=True)" > $O/build.log 2>&1
echo ALL DONE
