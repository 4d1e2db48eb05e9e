#!/usr/bin/env python
"""Diagnostic: two processes, one GPU each, issue mismatched collectives
(rank 0 one whole-model all-reduce, rank 1 the pipelined step's first
piece).  Prints per-rank timestamps of the call, the synchronize and the
status, to see which wait (if any) runs into the device timeout.

Round 2 ran this with both ranks on one GPU (profiles/r2_diag_piece_mismatch.txt);
since then ranks whose kernels wait on one another are never time-sliced on
one GPU (B200_PROFILING.md), so it needs two GPUs.  The same fault is covered
on one GPU by tests/test_gpu_emulated.py (CMN_TEST_EMUL_MISMATCH_RANK)."""
import os
import socket
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, port, timeout_ms):
    import torch
    import torch.distributed as dist

    import synth
    from paper_1908_00213_b200 import cmn
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    shapes = synth.mlp_shapes()
    comm = cmn.Comm.init(rank, 2, rank, dist.group.WORLD)
    comm.set_timeout(timeout_ms)
    w = [torch.from_numpy(p).cuda() for p in synth.params(shapes)]
    comm.register_params(w)
    comm.set_algo("twoshot")
    comm.set_pipeline(1 + rank)
    g = [torch.from_numpy(x).cuda() for x in synth.grads(shapes, workers=2)[rank]]
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.time()
    comm.step(g, "fp32", 0.1, 0.9)
    t1 = time.time()
    torch.cuda.synchronize()
    t2 = time.time()
    try:
        comm.poll_error()
        st = "OK"
    except cmn.CmnError as e:
        st = e.status_name
    print(f"rank {rank}: issue {t1 - t0:.3f}s sync {t2 - t1:.3f}s status {st}", flush=True)
    dist.barrier()
    comm.finalize()
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        raise SystemExit("needs 2 GPUs (ranks are never time-sliced on one GPU)")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    tmo = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=worker, args=(r, port, tmo)) for r in range(2)]
    t = time.time()
    for p in ps:
        p.start()
    for p in ps:
        p.join()
    print(f"total {time.time() - t:.1f}s")
