#!/bin/bash
# Round 2, session 3: the emulated world (barriers live in one cooperative
# launch) and the whole GPU suite with the multi-rank-on-one-GPU tests
# skipped; smoke.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; tail -30 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_emulated.py -m gpu -x -q -p no:cacheprovider --durations=10 > $O/r2s3_emulated.txt 2>&1; echo "emulated rc=$?" >> $O/r2s3_emulated.txt
tail -3 $O/r2s3_emulated.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rs --durations=15 --deselect tests/test_gpu_emulated.py > $O/r2s3_pytest_gpu.txt 2>&1; echo "suite rc=$?" >> $O/r2s3_pytest_gpu.txt
tail -3 $O/r2s3_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2s3_smoke.txt 2>&1; echo "smoke rc=$?" >> $O/r2s3_smoke.txt
tail -2 $O/r2s3_smoke.txt
