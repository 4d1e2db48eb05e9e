#!/bin/bash
# Round-2 call 5: sanitizers over the round-2 code (memcheck / initcheck /
# synccheck / racecheck on the parity suite, memcheck on the IPC suite incl.
# the fault-path tests), then the multi-process IPC suite under MPS (truly
# concurrent kernels of different processes, if the box has the daemon).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for tool in memcheck initcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all python -m pytest tests/test_gpu_parity.py -m 'gpu and not slow' -q -p no:cacheprovider > $O/san_${tool}_parity.txt 2>&1; echo "rc=$?" >> $O/san_${tool}_parity.txt
done
timeout 1200 compute-sanitizer --tool memcheck --target-processes all python -m pytest tests/test_gpu_ipc.py -m 'gpu and not slow' -q -p no:cacheprovider > $O/san_memcheck_ipc.txt 2>&1; echo "rc=$?" >> $O/san_memcheck_ipc.txt
# MPS probe
{
  which nvidia-cuda-mps-control || echo "no nvidia-cuda-mps-control"
  export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
  mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
  if which nvidia-cuda-mps-control; then
    nvidia-cuda-mps-control -d && echo "MPS daemon started"
    sleep 2
    timeout 900 python -m pytest tests/test_gpu_ipc.py -m gpu -q -p no:cacheprovider --timeout 300 -k "multiprocess_parity or cuda_graph or fused_allgather or sharded or slow_peer or stress or r50_full" 2>&1 | tail -30
    echo "pytest under MPS rc=${PIPESTATUS[0]}"
    echo quit | nvidia-cuda-mps-control
    sleep 2
    cat /tmp/mps_log/control.log 2>/dev/null | tail -5
  fi
} > $O/mps_probe.txt 2>&1
echo ALL DONE
# pack -> Adam-from-packed interplay (the 256-bit pack makes the following
# Adam update ~9 us slower at N = 1 in the back-to-back kernel bench): per
# kernel DRAM bytes and duration with the L2 state kept (--cache-control none)
for v in "-" "-DCMN_PACK_V8=0"; do
  if [ "$v" = "-" ]; then unset CMN_EXTRA_NVFLAGS; tag=v8; else export CMN_EXTRA_NVFLAGS="$v"; tag=v4; fi
  python -c "from paper_1908_00213_b200 import build; build.build(force=True)" > /dev/null 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum \
      --cache-control none --clock-control none -k regex:"k_pack|k_update_adam|k_update_sgd" -s 6 -c 6 --csv \
      --log-file $O/ncu_pack_then_update_$tag.csv python scripts/prof_driver.py --mode adam --iters 6 > /dev/null 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum \
      --cache-control none --clock-control none -k regex:"k_pack|k_update_sgd" -s 6 -c 6 --csv \
      --log-file $O/ncu_pack_then_sgd_$tag.csv python scripts/prof_driver.py --mode n1 --iters 6 > /dev/null 2>&1
done
unset CMN_EXTRA_NVFLAGS
python -c "from paper_1908_00213_b200 import build; build.build(force=True)" > /dev/null 2>&1
echo ALL DONE 2
