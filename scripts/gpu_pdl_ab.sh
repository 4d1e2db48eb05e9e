#!/bin/bash
# A/B of programmatic dependent launch for the N = 1 direct update (CMN_PDL).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
CMN_PDL=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "full_size_n1 or n1_direct or host_packed or kernel_timing or launch_count" > $O/pytest_pdl.log 2>&1; echo rc=$? >> $O/pytest_pdl.log
rm -f $O/pdl_ab.jsonl
for rep in 1 2 3; do for p in 0 1; do
  CMN_PDL=$p timeout 300 python bench.py --steps 200 --no-cpu-baseline 2>/dev/null | python -c "
import json, sys
d = json.loads(sys.stdin.read()); print(json.dumps({'pdl': $p, 'rep': $rep, 'us': d['value'], 'frac': d['roofline']['frac'], 'e2e_us': d['e2e']['value'], 'sm_mhz': d['clocks']['sm_mhz']}))" >> $O/pdl_ab.jsonl
done; done
echo ALL DONE
