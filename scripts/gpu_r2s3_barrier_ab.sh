#!/bin/bash
# Round 2, session 3: barrier memory-ordering variants (CMN_BARRIER_VARIANT
# 0 / 1 / 2, cmn_device.cuh) -- small all-reduce latency in the emulated
# world (graph replay), the emulated tests per variant, and an ncu launch
# list (gpu__time_duration) of the all-reduce kernels per variant.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
rm -f $O/barrier_ab.jsonl $O/barrier_ab_ncu_v*.csv
for rep in 1 2; do for v in ${VARIANTS:-0 1 2}; do
  export CMN_EXTRA_NVFLAGS="-DCMN_BARRIER_VARIANT=$v"
  python -c "from paper_1908_00213_b200 import build; build.build(force=True)" > $O/build_v$v.log 2>&1 || { echo "build $v failed"; continue; }
  timeout 600 python scripts/barrier_latency.py --variant v$v >> $O/barrier_ab.jsonl 2>> $O/barrier_ab.err
  if [ $rep = 1 ]; then
    timeout 900 python -m pytest tests/test_gpu_emulated.py -m gpu -q -p no:cacheprovider -k "not r50" > $O/barrier_ab_tests_v$v.txt 2>&1; echo "tests v$v rc=$?"
    CMD="python scripts/barrier_latency.py --worlds 8 --elems 256 --calls 4 --reps 2 --variant v$v"
    timeout 300 $CMD > /dev/null 2>&1 && \
      timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_oneshot|k_twoshot" \
        --csv --log-file $O/barrier_ab_ncu_v$v.csv $CMD > /dev/null 2>&1; echo "ncu v$v rc=$?"
  fi
done; done
unset CMN_EXTRA_NVFLAGS
python -c "from paper_1908_00213_b200 import build; build.build(force=True)" > $O/build.log 2>&1
echo ALL DONE
