#!/bin/bash
# Quick GPU iteration: build, GPU tests (optional), kernel bench, bench.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || echo "BUILD FAILED" >> $O/build.log
if [ -z "$SKIP_TESTS" ]; then
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 600 ${PYTEST_ARGS:-} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
fi
timeout 900 python scripts/kernel_bench.py --worlds ${WORLDS:-1,8} > $O/kernel_bench.jsonl 2> $O/kernel_bench.err
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
for c in ${EXTRA:-}; do eval "$c"; done
echo ALL DONE
