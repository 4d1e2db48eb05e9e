#!/bin/bash
# ncu --set full captures of the step's kernels (one GPU, simulated N for the all-reduce).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for k in k_pack k_update_sgd k_update_direct; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o $O/prof_$k -f python scripts/prof_driver.py --mode n1 > $O/prof_$k.log 2>&1
done
for k in k_twoshot k_oneshot; do
  a=${k#k_}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 9 -c 1 \
      -o $O/prof_${k}_sim8 -f python scripts/prof_driver.py --mode sim8 --algo $a > $O/prof_$k.log 2>&1
done
echo ALL DONE
