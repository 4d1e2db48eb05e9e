#!/bin/bash
# A/B of programmatic dependent launch for k_pack / k_update_sgd (CMN_PDL),
# plus the full GPU suite with PDL on.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || echo "BUILD FAILED" >> $O/build.log
rm -f $O/pdl2_ab.jsonl
for rep in ${REPS:-1 2}; do for p in 0 1; do
  CMN_PDL=$p timeout 600 python scripts/kernel_bench.py --worlds ${WORLDS:-1,8} 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); d['pdl'] = $p; d['rep'] = $rep; print(json.dumps(d))" >> $O/pdl2_ab.jsonl
done; done
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
echo ALL DONE
