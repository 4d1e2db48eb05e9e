#!/bin/bash
# A/B of k_adam_direct variants (build switches CMN_ADAM_DIRECT_CS, CMN_ADAM_PASSES).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out; rm -f gpurun_out/adam_ab.jsonl
for rep in 1 2; do for cfg in "-DCMN_ADAM_PASSES=2" "-DCMN_ADAM_PASSES=1" "-DCMN_ADAM_PASSES=4"; do
  export CMN_EXTRA_NVFLAGS="$cfg"
  python -c "from paper_1908_00213_b200 import build; build.build(force=True)" > gpurun_out/b.log 2>&1
  timeout 300 python scripts/kernel_bench.py --worlds 1 2>/dev/null | python -c "
import json, sys
for l in sys.stdin:
    d = json.loads(l); print(json.dumps({'cfg': '$cfg', 'rep': $rep, 'dtype': d['dtype'], 'adam_step_us': d['adam_step_us'], 'adam_update_us': d['adam_update_us']}))" >> gpurun_out/adam_ab.jsonl
done; done
unset CMN_EXTRA_NVFLAGS
