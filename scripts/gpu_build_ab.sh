#!/bin/bash
# Generic build-switch A/B on one box: for each variant in $VARIANTS (flag
# sets separated by ';', "-" = default build), rebuild libcmn.so with
# CMN_EXTRA_NVFLAGS and run scripts/kernel_bench.py --worlds $WORLDS; REPS
# alternating repetitions.  Output: gpurun_out/build_ab.jsonl (variant, rep, record).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
rm -f $O/build_ab.jsonl
IFS=';' read -ra VS <<< "${VARIANTS:--}"
for rep in $(seq 1 ${REPS:-2}); do for v in "${VS[@]}"; do
  if [ "$v" = "-" ]; then unset CMN_EXTRA_NVFLAGS; else export CMN_EXTRA_NVFLAGS="$v"; fi
  python -c "from paper_1908_00213_b200 import build; build.build(force=True)" > $O/build_ab_build.log 2>&1 || echo "build failed: $v" >> $O/build_ab.err
  timeout 600 python scripts/kernel_bench.py --worlds ${WORLDS:-1} 2>>$O/build_ab.err | python -c "
import json, sys
for l in sys.stdin:
    d = json.loads(l); d['variant'] = '''$v'''; d['rep'] = $rep; print(json.dumps(d))" >> $O/build_ab.jsonl
done; done
unset CMN_EXTRA_NVFLAGS
python -c "from paper_1908_00213_b200 import build; build.build(force=True)" > $O/build.log 2>&1
echo ALL DONE
