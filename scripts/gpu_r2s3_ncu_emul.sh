#!/bin/bash
# Round 2, session 3: ncu --set full of the emulated N = 8 fp32 two-shot with
# the one-fence barrier (compare r2s3_ncu_k_twoshot_emul8.json, the round-2
# barrier), after the same command ran clean.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
CMD="python scripts/emulated_bench.py --worlds 8 --algos twoshot --iters 3"
timeout 300 $CMD > $O/r2s3_emul_plain2.jsonl 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_twoshot -c 1 \
  -o $O/r2s3_k_twoshot_emul8_onefence $CMD > $O/r2s3_ncu2.log 2>&1; echo "ncu rc=$?"
tail -3 $O/r2s3_ncu2.log
