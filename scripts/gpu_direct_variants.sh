#!/bin/bash
# A/B of the N = 1 direct-update kernel designs (CMN_DIRECT_VARIANT 0/1/2):
# parity of each, then alternating bench runs.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for v in 0 1 2; do
  CMN_DIRECT_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "full_size_n1 or n1_direct or host_packed or launch_count or kernel_timing" > $O/pytest_var$v.log 2>&1; echo rc=$? >> $O/pytest_var$v.log
done
rm -f $O/direct_variants.jsonl
for rep in 1 2 3; do for v in 0 1 2; do
  CMN_DIRECT_VARIANT=$v timeout 300 python bench.py --steps 200 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'variant': $v, 'rep': $rep, 'us': d['value'], 'frac': d['roofline']['frac'], 'sm_mhz': d['clocks']['sm_mhz']}))" >> $O/direct_variants.jsonl
done; done
echo ALL DONE
