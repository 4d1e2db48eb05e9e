#!/bin/bash
# Build-switch A/B on the N = 1 bench line: for each variant in $VARIANTS
# (';'-separated flag sets, "-" = default build) rebuild libcmn.so and run
# bench.py (100 steps): back-to-back value, per-step median, isolated launch.
# REPS alternating repetitions -> gpurun_out/bench_build_ab.jsonl.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
rm -f $O/bench_build_ab.jsonl
IFS=';' read -ra VS <<< "${VARIANTS:--}"
for rep in $(seq 1 ${REPS:-3}); do for v in "${VS[@]}"; do
  if [ "$v" = "-" ]; then unset CMN_EXTRA_NVFLAGS; else export CMN_EXTRA_NVFLAGS="$v"; fi
  python -c "from paper_1908_00213_b200 import build; build.build(force=True)" > /dev/null 2>&1 || echo "build failed: $v" >> $O/bench_build_ab.err
  timeout 300 python bench.py --steps 100 --warmup 20 --no-cpu-baseline --no-e2e --dtype ${DTYPE:-fp32} 2>>$O/bench_build_ab.err | python -c "
import json, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1]); r = d['roofline']
print(json.dumps({'variant': '''$v''', 'rep': $rep, 'us': d['value'], 'per_step_median_us': d['details']['per_step_us']['median_us'],
      'isolated_us': r['kernel_us_per_launch_isolated'], 'sm_mhz': d['clocks']['sm_mhz']}))" >> $O/bench_build_ab.jsonl
done; done
unset CMN_EXTRA_NVFLAGS
python -c "from paper_1908_00213_b200 import build; build.build(force=True)" > /dev/null 2>&1
echo ALL DONE
