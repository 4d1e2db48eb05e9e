#!/bin/bash
# A/B of items per CTA in the library's pack kernel (build switch CMN_PACK_ITEMS).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
rm -f $O/pack_ab.jsonl
for rep in 1 2; do for k in 1 2 4; do
  export CMN_EXTRA_NVFLAGS=-DCMN_PACK_ITEMS=$k
  python -c "from paper_1908_00213_b200 import build; build.build(force=True)" > $O/build_pack$k.log 2>&1
  timeout 300 python scripts/kernel_bench.py --worlds 1 2>/dev/null | python -c "
import json, sys
for l in sys.stdin:
    d = json.loads(l); print(json.dumps({'items_per_cta': $k, 'rep': $rep, 'dtype': d['dtype'], 'pack_us': d['allreduce_incl_pack_us'], 'pack_gbs': d['pack_gbs']}))" >> $O/pack_ab.jsonl
done; done
unset CMN_EXTRA_NVFLAGS
python -c "from paper_1908_00213_b200 import build; build.build(force=True)" > $O/build.log 2>&1
echo ALL DONE
