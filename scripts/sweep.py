#!/usr/bin/env python
"""BASELINE config 5: packed-buffer sweep, 64 KB .. 1 GB, fp32/fp16, of the
hand-written P2P all-reduce (one-shot, two-shot, auto) against NCCL
(PAPER.md:480-486 names NCCL as ChainerMN's primary all-reduce library).

    torchrun --nproc-per-node N scripts/sweep.py [--max-mb 1024]
    python scripts/sweep.py --sim 8          # mechanics only: local HBM, no NVLink

One flat "tensor" of S bytes is registered; each point times
cmn_allreduce_grads (pack + all-reduce) over --iters calls after warm-up,
max over ranks.  Output: one JSON line per (algo, dtype, bytes) with
latency, algBW = S/t and busBW = 2(N-1)/N * S/t, plus SPEC-style CSV
columns (n, bytes, comm_ms_mean, iter_ms_mean).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1908_00213_b200 import CmnError, Comm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sim", type=int, default=0)
    ap.add_argument("--min-kb", type=int, default=64)
    ap.add_argument("--max-mb", type=int, default=1024)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--algos", default="oneshot,twoshot,auto,nccl")
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > torch.cuda.device_count():   # never time-slice barrier ranks on one GPU
        raise SystemExit(f"{world} ranks need {world} GPUs (B200_PROFILING.md)")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    n = a.sim if a.sim else world
    sizes = []
    s = a.min_kb << 10
    while s <= a.max_mb << 20:
        sizes.append(s)
        s *= 2
    for dtype, esz in (("fp32", 4), ("fp16", 2)):
        for nbytes in sizes:
            elems = nbytes // esz
            comm = Comm.simulated_world(a.sim) if a.sim else Comm.init(
                rank, world, local, dist.group.WORLD if world > 1 else None)
            w = [torch.zeros(elems, dtype=torch.float32, device="cuda")]
            comm.register_params(w)
            gw = [[torch.randn(elems, device="cuda")] for _ in range(n if a.sim else 1)]
            table = comm.prepare(gw if a.sim else gw[0])
            for algo in a.algos.split(","):
                try:
                    comm.set_algo(algo)
                except CmnError as e:
                    if rank == 0:
                        print(json.dumps({"algo": algo, "skipped": str(e)}), flush=True)
                    continue
                for _ in range(a.warmup):
                    comm.allreduce_grads(table, dtype)
                torch.cuda.synchronize()
                if world > 1:
                    dist.barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(a.iters):
                    comm.allreduce_grads(table, dtype)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / a.iters
                if world > 1:
                    t = torch.tensor([ms], dtype=torch.float64)
                    dist.all_reduce(t, op=dist.ReduceOp.MAX)
                    ms = float(t.item())
                S = elems * esz
                if rank == 0:
                    print(json.dumps({"n": n, "simulated": bool(a.sim), "algo": algo, "dtype": dtype,
                                      "bytes": S, "us": ms * 1e3, "alg_gbs": S / (ms * 1e-3) / 1e9,
                                      "bus_gbs": 2 * (n - 1) / n * S / (ms * 1e-3) / 1e9 if n > 1 else None,
                                      "csv": f"{n},{S},{ms:.6f},{ms:.6f}"}), flush=True)
            comm.finalize()
            del w, gw, table
            torch.cuda.empty_cache()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
