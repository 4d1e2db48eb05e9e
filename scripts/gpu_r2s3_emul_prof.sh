#!/bin/bash
# Round 2, session 3: emulated-world all-reduce timings (barriers live, one
# cooperative launch, local HBM) and one ncu --set full capture of the
# emulated N = 8 fp32 two-shot launch.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; tail -30 $O/build.log; exit 1; }
timeout 900 python scripts/emulated_bench.py --worlds 2,4,8 > $O/r2s3_emulated_bench.jsonl 2> $O/r2s3_emulated_bench.err; echo "bench rc=$?"
cat $O/r2s3_emulated_bench.jsonl
CMD="python scripts/emulated_bench.py --worlds 8 --algos twoshot --iters 3"
timeout 300 $CMD > $O/r2s3_emul_plain.jsonl 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_twoshot -c 1 \
  -o $O/r2s3_k_twoshot_emul8 $CMD > $O/r2s3_ncu.log 2>&1; echo "ncu rc=$?"
tail -5 $O/r2s3_ncu.log
