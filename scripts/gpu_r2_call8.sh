#!/bin/bash
# Round-2 call 8: the poison-flag barrier -- mismatch diagnostic x3, the IPC
# suite, the new parity tests (16-B aligned pack fallback, division through
# every kernel), memcheck over the IPC fault-path tests.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for i in 1 2 3; do timeout 300 python scripts/diag_piece_mismatch.py 20000 >> $O/diag_mismatch.txt 2>&1; done
timeout 1800 python -m pytest tests/test_gpu_ipc.py tests/test_gpu_parity.py -m gpu -q --timeout 900 -p no:cacheprovider --durations=10 > $O/pytest_ipc_parity.log 2>&1; echo "pytest rc=$?" >> $O/pytest_ipc_parity.log
timeout 900 compute-sanitizer --tool memcheck --target-processes all python -m pytest tests/test_gpu_ipc.py -m gpu -q -p no:cacheprovider -k "skipped or mismatch or slow_peer" > $O/san_memcheck_faults.txt 2>&1; echo "rc=$?" >> $O/san_memcheck_faults.txt
echo ALL DONE
