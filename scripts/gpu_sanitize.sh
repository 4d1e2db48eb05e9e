#!/bin/bash
# compute-sanitizer memcheck + synccheck over the GPU parity suite (current kernels).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 compute-sanitizer --tool memcheck --target-processes all python -m pytest tests/test_gpu_parity.py -m 'gpu and not slow' -q -p no:cacheprovider > $O/memcheck.txt 2>&1; echo "rc=$?" >> $O/memcheck.txt
timeout 1500 compute-sanitizer --tool synccheck --target-processes all python -m pytest tests/test_gpu_parity.py -m 'gpu and not slow' -q -p no:cacheprovider > $O/synccheck.txt 2>&1; echo "rc=$?" >> $O/synccheck.txt
timeout 900 compute-sanitizer --tool memcheck --target-processes all python -m pytest tests/test_gpu_ipc.py -m 'gpu and not slow' -q -p no:cacheprovider -x > $O/memcheck_ipc.txt 2>&1; echo "rc=$?" >> $O/memcheck_ipc.txt
echo ALL DONE
