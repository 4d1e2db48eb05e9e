#!/bin/bash
# compute-sanitizer racecheck (shared-memory data hazards) over the GPU parity
# suite: SURVEY §4 asks for memcheck, racecheck and synccheck of the kernels.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 2400 compute-sanitizer --tool racecheck --racecheck-report all --target-processes all \
    python -m pytest tests/test_gpu_parity.py -m 'gpu and not slow' -q -p no:cacheprovider > $O/racecheck.txt 2>&1
echo "rc=$?" >> $O/racecheck.txt
echo ALL DONE
