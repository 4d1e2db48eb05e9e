#!/bin/bash
# PyTorch multi-tensor optimizers vs cmn_step / cmn_step_adam at N = 1 (3 alternating reps).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
rm -f $O/torch_optim_ref.jsonl
for r in 1 2 3; do
  timeout 600 python scripts/torch_optim_reference.py >> $O/torch_optim_ref.jsonl 2>> $O/torch_optim_ref.err
done
echo ALL DONE
