#!/bin/bash
# A/B of the N = 1 direct kernel's launch order of work items (CMN_ITEM_ORDER
# 1 = full items first then partial ones by decreasing length, 0 =
# registration order): bench back to back, per-step median, isolated launch;
# 3 alternating runs each, fp32.  Plus the parity tests of the direct path.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_benched.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "n1 or direct or step_adam or launch_count or kernel_timing" > $O/pytest_order.log 2>&1; echo "rc=$?" >> $O/pytest_order.log
rm -f $O/order_ab.jsonl
for rep in 1 2 3; do for o in 1 0; do
  CMN_ITEM_ORDER=$o timeout 300 python bench.py --steps 100 --warmup 20 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1]); r = d['roofline']
print(json.dumps({'item_order': $o, 'rep': $rep, 'us': d['value'], 'per_step_median_us': d['details']['per_step_us']['median_us'],
      'isolated_us': r['kernel_us_per_launch_isolated'], 'flushed_us': d['details']['step_us_after_l2_write_flush'], 'sm_mhz': d['clocks']['sm_mhz']}))" >> $O/order_ab.jsonl
done; done
echo ALL DONE
