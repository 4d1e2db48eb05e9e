#!/bin/bash
# Round-2 call 6: the whole GPU suite (durations), smoke, the IPC suite under
# MPS with per-client SM limits (truly concurrent kernels of different
# processes), the N = 1 bench fp32 / fp16.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/build_smoke.log 2>&1 || echo "BUILD/SMOKE FAILED" >> $O/build_smoke.log
timeout 2700 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider --durations=25 > $O/pytest_gpu_full.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_full.log
timeout 600 python bench.py --steps 100 --warmup 20 > $O/bench_fp32.json 2> $O/bench_fp32.err
timeout 600 python bench.py --steps 100 --warmup 20 --dtype fp16 > $O/bench_fp16.json 2> $O/bench_fp16.err
{
  export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
  mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
  nvidia-cuda-mps-control -d && echo "MPS daemon started"
  sleep 2
  # every client limited to 12 % of the SMs: up to 8 ranks' barrier grids are
  # co-resident on the one GPU (on separate GPUs each rank has all its SMs)
  export CUDA_MPS_ACTIVE_THREAD_PERCENTAGE=12
  timeout 1800 python -m pytest tests/test_gpu_ipc.py tests/test_gpu_autograd.py -m gpu -q -p no:cacheprovider --timeout 600 -k "ipc or processes" 2>&1 | tail -15
  echo "pytest under MPS rc=${PIPESTATUS[0]}"
  echo quit | nvidia-cuda-mps-control
  sleep 2
} > $O/mps_ipc.txt 2>&1
echo ALL DONE
