#!/bin/bash
# Round 2, session 3 validation: the whole GPU suite (simulated + emulated
# worlds), smoke, the driver's bench command and the reference arm.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; tail -30 $O/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2s3v_smoke.txt 2>&1; echo "smoke rc=$?" >> $O/r2s3v_smoke.txt
tail -2 $O/r2s3v_smoke.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rs --durations=20 > $O/r2s3v_pytest_gpu.txt 2>&1; echo "suite rc=$?" >> $O/r2s3v_pytest_gpu.txt
tail -4 $O/r2s3v_pytest_gpu.txt
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/r2s3v_bench.json 2> $O/r2s3v_bench.err; echo "bench rc=$?"
tail -c 600 $O/r2s3v_bench.json
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/r2s3v_bench_ref.json 2> $O/r2s3v_bench_ref.err; echo "ref rc=$?"
timeout 900 python scripts/emulated_bench.py --worlds 2,4,8 --algos twoshot > $O/r2s3v_emulated_bench.jsonl 2>/dev/null; echo "emul rc=$?"
