#!/bin/bash
# Round-2 iteration on the GPU box: build, the selected GPU tests (slow ones
# included), kernel bench at N = 1 and simulated N = 8, the N = 1 bench line.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || echo "BUILD FAILED" >> $O/build.log
timeout ${TEST_TIMEOUT:-2400} python -m pytest ${TESTS:-tests} -m gpu -q -x --timeout 900 -p no:cacheprovider ${PYTEST_ARGS:-} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
if [ -z "$SKIP_KBENCH" ]; then
timeout 900 python scripts/kernel_bench.py --worlds ${WORLDS:-1,8} > $O/kernel_bench.jsonl 2> $O/kernel_bench.err
fi
if [ -z "$SKIP_BENCH" ]; then
timeout 600 python bench.py ${BENCH_ARGS:-} > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
fi
for c in ${EXTRA:-}; do eval "$c"; done
echo ALL DONE
