#!/bin/bash
# BASELINE config 4 sweep with the calibrated, interleaved-median overlap_bench:
# bucket size x stream-kernel grid cap (cmn_set_stream_ctas) x GEMM SM carveout,
# N = 1 real communicator and 8 simulated ranks; then the parity tests of the
# capped grids and a default-grid kernel bench (no regression).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "stream_ctas or adam or bucket or n1 or fused or value_sets" > $O/pytest_sc.log 2>&1; echo "rc=$?" >> $O/pytest_sc.log
timeout 600 python scripts/kernel_bench.py --worlds 1 > $O/kernel_bench.jsonl 2> $O/kernel_bench.err
rm -f $O/overlap_sweep.jsonl
for mb in ${MBS:-4 8 16 25}; do
  for sc in ${SCS:-0 16 32 64 148 296}; do
    for co in ${COS:-0 32}; do
      timeout 600 python scripts/overlap_bench.py --bwd-ms 1.0 --bucket-mb $mb --stream-ctas $sc --carveout $co >> $O/overlap_sweep.jsonl 2>> $O/overlap_sweep.err
    done
  done
done
for mb in 4 25; do for sc in 0 64; do
  timeout 600 python scripts/overlap_bench.py --sim 8 --bwd-ms 4.0 --bucket-mb $mb --stream-ctas $sc --ar-ctas 64 >> $O/overlap_sweep.jsonl 2>> $O/overlap_sweep.err
done; done
echo ALL DONE
