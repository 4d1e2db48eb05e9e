#!/bin/bash
# Round 2, session 3: barrier variants at large sizes (emulated R50
# all-reduce, scripts/emulated_bench.py) and the small-size latency incl. the
# diagnostic gpu-scope variant 5.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
rm -f $O/barrier_ab2.jsonl $O/barrier_ab2_r50.jsonl
for rep in 1 2; do for v in 0 3 5; do
  export CMN_EXTRA_NVFLAGS="-DCMN_BARRIER_VARIANT=$v"
  python -c "from paper_1908_00213_b200 import build; build.build(force=True)" > $O/build_v$v.log 2>&1 || { echo "build $v failed"; continue; }
  timeout 600 python scripts/barrier_latency.py --variant v$v --worlds 2,8 --elems 256 >> $O/barrier_ab2.jsonl 2>> $O/barrier_ab2.err
  timeout 600 python scripts/emulated_bench.py --worlds 8 --iters 10 | python -c "
import json, sys
for l in sys.stdin:
    d = json.loads(l); d['variant'] = 'v$v'; d['rep'] = $rep; print(json.dumps(d))" >> $O/barrier_ab2_r50.jsonl
done; done
unset CMN_EXTRA_NVFLAGS
python -c "from paper_1908_00213_b200 import build; build.build(force=True)" > $O/build.log 2>&1
echo ALL DONE
