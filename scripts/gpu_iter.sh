#!/bin/bash
# Iteration check: build, a pytest selection (PYTEST_K), and the N = 2 bench
# under torchrun with both ranks on the one GPU (mechanics only).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || echo "BUILD FAILED" >> $O/build.log
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 ${PYTEST_K:+-k "$PYTEST_K"} > $O/pytest_iter.log 2>&1; echo "pytest rc=$?" >> $O/pytest_iter.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
    bench.py --gpus 2 --steps 10 --warmup 3 --min-warmup-s 0 --no-cpu-baseline > $O/bench_n2_1gpu.json 2> $O/bench_n2_1gpu.err
echo "torchrun rc=$?" >> $O/bench_n2_1gpu.err
for c in "${EXTRA[@]}"; do eval "$c"; done
echo ALL DONE
