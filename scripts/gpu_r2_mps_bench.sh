#!/bin/bash
# The N > 1 bench path end to end with truly concurrent ranks (MPS on the
# one GPU, 100/N % of the SMs per rank): torchrun N = 2 and 4.  The numbers
# are one GPU's HBM shared by N ranks, not NVLink; the point is that every
# phase (collective autotune, graph capture, comparisons, timed region,
# kernel timing, replica check, e2e, config-5 sweep) completes concurrently.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d
sleep 2
for n in 2 4; do
  CUDA_MPS_ACTIVE_THREAD_PERCENTAGE=$((100 / n)) timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
      --master-addr 127.0.0.1 --master-port $((29700 + n)) bench.py --gpus $n --steps 20 --warmup 5 \
      > $O/mps_bench_n$n.json 2> $O/mps_bench_n$n.err
  echo "n=$n rc=$?" >> $O/mps_bench_rc.txt
done
echo quit | nvidia-cuda-mps-control
echo ALL DONE
