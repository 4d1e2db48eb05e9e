#!/bin/bash
# A/B of the streaming cache hints (.cs) in the pack / update / all-reduce
# kernels: kernel bench at N = 1 and simulated N = 8 with the default build,
# then with -DCMN_NO_STREAMING_HINTS, twice each (alternating).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
rm -f $O/hints_ab.jsonl
for rep in 1 2; do for mode in cs plain; do
  if [ $mode = plain ]; then export CMN_EXTRA_NVFLAGS=-DCMN_NO_STREAMING_HINTS; else unset CMN_EXTRA_NVFLAGS; fi
  python -c "from paper_1908_00213_b200 import build; build.build(force=True)" > $O/build_$mode.log 2>&1
  timeout 600 python scripts/kernel_bench.py --worlds 1,8 2>/dev/null | python -c "
import json, sys
for l in sys.stdin:
    d = json.loads(l); d['hints'] = '$mode'; d['rep'] = $rep; print(json.dumps(d))" >> $O/hints_ab.jsonl
  timeout 300 python bench.py --steps 200 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json, sys
d = json.loads(sys.stdin.read()); print(json.dumps({'hints': '$mode', 'rep': $rep, 'bench_us': d['value']}))" >> $O/hints_ab.jsonl
done; done
unset CMN_EXTRA_NVFLAGS
python -c "from paper_1908_00213_b200 import build; build.build(force=True)" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > $O/pytest_parity.log 2>&1; echo rc=$? >> $O/pytest_parity.log
echo ALL DONE
