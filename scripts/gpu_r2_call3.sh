#!/bin/bash
# Round-2 call 3: parity (division templates), pack/direct 256-bit A/B,
# negative control of the one-shot end barrier, new bench lines.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/build_smoke.log 2>&1 || echo "BUILD/SMOKE FAILED" >> $O/build_smoke.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench.py -m gpu -q -x --timeout 900 -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
# negative control: without the end barrier the slow-peer test is expected to FAIL
CMN_TEST_NO_END_BARRIER=1 timeout 600 python -m pytest tests/test_gpu_ipc.py -k slow_peer -m gpu -q --timeout 300 -p no:cacheprovider > $O/negative_control_no_end_barrier.log 2>&1; echo "rc=$? (nonzero expected)" >> $O/negative_control_no_end_barrier.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_reference.json 2> $O/bench_reference.err
VARIANTS="-;-DCMN_PACK_V8=0;-DCMN_DIRECT_V8=1" REPS=2 WORLDS=1 bash scripts/gpu_build_ab.sh
echo ALL DONE
