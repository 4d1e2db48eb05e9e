#!/bin/bash
# e2e (host-buffer step) iteration: parity tests, then bench.py's e2e under
# the read-back modes (SM stores vs copy engine) and piece plans.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "step_host" > gpurun_out/pytest_e2e.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_e2e.log
for zc in 1 0; do for p in "" 4 8 16; do
  CMN_E2E_ZC=$zc CMN_E2E_PIECES=$p timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_e2e_zc${zc}_p$p.json 2>/dev/null
done; done
echo DONE
