#!/bin/bash
# A/B of work-item size and CTA size (build switches CMN_ITEM_ELEMS, CMN_THREADS).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out; rm -f gpurun_out/item_size_ab.jsonl
for rep in 1 2; do for cfg in "" "-DCMN_ITEM_ELEMS=8192 -DCMN_THREADS=512" "-DCMN_ITEM_ELEMS=8192" "-DCMN_ITEM_ELEMS=2048 -DCMN_THREADS=128"; do
  export CMN_EXTRA_NVFLAGS="$cfg"
  python -c "from paper_1908_00213_b200 import build; build.build(force=True)" > gpurun_out/b.log 2>&1
  timeout 300 python bench.py --steps 200 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json, sys
d = json.loads(sys.stdin.read()); print(json.dumps({'cfg': '$cfg', 'rep': $rep, 'bench_us': d['value']}))" >> gpurun_out/item_size_ab.jsonl
  timeout 300 python scripts/kernel_bench.py --worlds 1 2>/dev/null | python -c "
import json, sys
for l in sys.stdin:
    d = json.loads(l); print(json.dumps({'cfg': '$cfg', 'rep': $rep, 'dtype': d['dtype'], 'pack_us': d['allreduce_incl_pack_us'], 'update_us': d['update_us'], 'adam_step_us': d['adam_step_us']}))" >> gpurun_out/item_size_ab.jsonl
done; done
unset CMN_EXTRA_NVFLAGS
python -c "from paper_1908_00213_b200 import build; build.build(force=True)" > gpurun_out/b.log 2>&1
