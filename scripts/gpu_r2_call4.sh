#!/bin/bash
# Round-2 call 4: pack 256-bit variants A/B, ncu of the v8 pack (both dtypes),
# the N = 8 time-sliced bench test.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
VARIANTS="-;-DCMN_PACK_V8=0;-DCMN_PACK_ITEMS=2;-DCMN_PACK_THREADS=128;-DCMN_PACK_THREADS=512" REPS=2 WORLDS=1 bash scripts/gpu_build_ab.sh
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for dt in fp32 fp16; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pack -s 2 -c 1 \
      -o $O/prof_k_pack_v8_$dt -f python scripts/prof_driver.py --mode n1 --dtype $dt > $O/prof_k_pack_v8_$dt.log 2>&1
done
timeout 1500 python -m pytest tests/test_gpu_bench.py -m gpu -q -x --timeout 1400 -p no:cacheprovider -k "n8 or same_config" > $O/pytest_bench.log 2>&1; echo "pytest rc=$?" >> $O/pytest_bench.log
echo ALL DONE
