#!/bin/bash
# Soak of the cross-process barrier protocol under MPS (the ranks' kernels
# truly concurrent on one GPU, 12 % of the SMs per client): the random-
# schedule stress test with 600 steps (schedule, algorithm and grid sizes
# redrawn every step), 2 and 3 ranks, bit-exact vs 600 oracle steps; then the
# whole IPC file twice more.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d && echo "MPS daemon started" > $O/soak.txt
sleep 2
export CUDA_MPS_ACTIVE_THREAD_PERCENTAGE=12
CMN_STRESS_STEPS=600 timeout 2400 python -m pytest tests/test_gpu_ipc.py -m gpu -q -p no:cacheprovider --timeout 2000 -k stress --durations=5 >> $O/soak.txt 2>&1; echo "stress-600 rc=$?" >> $O/soak.txt
for i in 1 2; do
  timeout 1200 python -m pytest tests/test_gpu_ipc.py -m gpu -q -p no:cacheprovider --timeout 600 >> $O/soak.txt 2>&1; echo "ipc pass $i rc=$?" >> $O/soak.txt
done
echo quit | nvidia-cuda-mps-control
echo ALL DONE
