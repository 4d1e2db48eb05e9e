#!/bin/bash
# A/B of the pack kernel's CTA size (build switch CMN_PACK_THREADS).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
rm -f $O/pack_threads_ab.jsonl
for rep in 1 2; do for t in 256 128 512 64; do
  export CMN_EXTRA_NVFLAGS=-DCMN_PACK_THREADS=$t
  python -c "from paper_1908_00213_b200 import build; build.build(force=True)" > $O/build_pt$t.log 2>&1
  timeout 300 python scripts/kernel_bench.py --worlds 1 2>/dev/null | python -c "
import json, sys
for l in sys.stdin:
    d = json.loads(l); print(json.dumps({'pack_threads': $t, 'rep': $rep, 'dtype': d['dtype'], 'pack_us': d['allreduce_incl_pack_us']}))" >> $O/pack_threads_ab.jsonl
done; done
export CMN_EXTRA_NVFLAGS=-DCMN_PACK_THREADS=128
python -c "from paper_1908_00213_b200 import build; build.build(force=True)" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "mlp_parity or ragged or edge_layouts or pipelined" > $O/pytest_pt.log 2>&1; echo rc=$? >> $O/pytest_pt.log
unset CMN_EXTRA_NVFLAGS
echo ALL DONE
