#!/bin/bash
# Round 2, session 3: compute-sanitizer memcheck over the emulated-world tests
# (the new cooperative all-reduce path: cta_rank mapping, per-rank epochs,
# fault injection).  One sanitizer tool per call (B200_PROFILING.md).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_emulated.py -m gpu -q -p no:cacheprovider -k "not r50" > $O/r2s3_emul_plain.txt 2>&1; echo "plain rc=$?" >> $O/r2s3_emul_plain.txt
tail -2 $O/r2s3_emul_plain.txt
timeout 2400 compute-sanitizer --tool memcheck --target-processes all --error-exitcode 99 \
  python -m pytest tests/test_gpu_emulated.py -m gpu -q -p no:cacheprovider -k "not r50" > $O/r2s3_memcheck_emulated.txt 2>&1
echo "memcheck rc=$?" >> $O/r2s3_memcheck_emulated.txt
tail -5 $O/r2s3_memcheck_emulated.txt
