#!/usr/bin/env python
"""The all-reduce kernels with the cross-rank barriers LIVE on one GPU:
cmn_init_emulated runs every rank's one-shot / two-shot as ONE cooperative
launch (block r * G + b = CTA b of rank r), so the flags, epochs and
mid / end barriers cost what they cost -- but every byte is local HBM
(there is no NVLink on a one-GPU box).  The kernel's device time (CUDA
events around each launch, cmn_set_kernel_timing) against the bytes the
emulated launch moves through HBM:

  two-shot: every rank reads the N copies of its chunk and writes it
            (N + 1) L c, then reads and writes the N - 1 other chunks
            2 (N - 1) L c  ->  (3N - 1) L c in all
  one-shot: every rank reads all N buffers and writes one: N (N + 1) L c

c = 4 (fp32) or 2 (fp16) bytes, L the padded length.  Prints one JSON line per
(N, dtype, algo), frac against MEASURED_PEAKS.json hbm_gbs.

    python scripts/emulated_bench.py [--worlds 2,4,8] [--iters 20]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1908_00213_b200 import Comm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--worlds", default="2,4,8")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--algos", default="twoshot,oneshot")
    ap.add_argument("--sweep", action="store_true",
                    help="config-5 sizes instead of R50: one flat fp32 tensor of 64 KB .. 256 MB, "
                         "pack + all-reduce per call (latency floor of the barrier kernels)")
    args = ap.parse_args()
    if args.sweep:
        return sweep(args)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    shapes = synth.resnet50_shapes()
    params0 = synth.params(shapes)
    dev = "cuda:0"
    for N in [int(x) for x in args.worlds.split(",")]:
        g = [[torch.from_numpy(x).to(dev) for x in gw] for gw in synth.grads(shapes, workers=N)]
        for dtype in ("fp32", "fp16"):
            c = 4 if dtype == "fp32" else 2
            for algo in args.algos.split(","):
                comm = Comm.emulated_world(N)
                try:
                    w = [torch.from_numpy(p.copy()).to(dev) for p in params0]
                    comm.register_params(w)
                    comm.set_algo(algo)
                    L = comm.layout()[1]
                    table = comm.prepare([x for gw in g for x in gw])
                    for _ in range(3):
                        comm.allreduce_grads(table, dtype)
                    torch.cuda.synchronize()
                    comm.set_kernel_timing(True)
                    for _ in range(args.iters):
                        comm.allreduce_grads(table, dtype)
                    torch.cuda.synchronize()
                    ms, n = comm.kernel_timing()
                    comm.set_kernel_timing(False)
                    comm.poll_error()
                    us = ms / n * 1e3
                    nbytes = ((3 * N - 1) if algo == "twoshot" else N * (N + 1)) * L * c
                    gbs = nbytes / (us * 1e-6) / 1e9
                    print(json.dumps({"what": "emulated all-reduce (one cooperative launch, barriers live)",
                                      "N": N, "dtype": dtype, "algo": algo, "launches": n,
                                      "kernel_us": us, "hbm_bytes": nbytes, "hbm_gbs": gbs,
                                      "frac": gbs / peak, "peak": peak}), flush=True)
                finally:
                    comm.finalize()
        del g
        torch.cuda.empty_cache()


def sweep(args):
    """Per-call device time of cmn_allreduce_grads (all ranks' packs + the
    one cooperative all-reduce launch) on one flat fp32 tensor per rank, S
    from 64 KB to 256 MB: at small S this is the latency floor of the
    barrier kernels without NVLink (launches + flag round trips through the
    one L2)."""
    dev = "cuda:0"
    stream = torch.cuda.current_stream()
    for N in [int(x) for x in args.worlds.split(",")]:
        for S in (64 << 10, 1 << 20, 16 << 20, 256 << 20):
            n = S // 4
            g = [torch.empty(n, device=dev).uniform_(-1e-2, 1e-2) for _ in range(N)]
            for algo in args.algos.split(","):
                comm = Comm.emulated_world(N)
                try:
                    w = torch.zeros(n, device=dev)
                    comm.register_params([w])
                    comm.set_algo(algo)
                    table = comm.prepare(g)
                    for _ in range(5):
                        comm.allreduce_grads(table, "fp32")
                    torch.cuda.synchronize()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    for _ in range(args.iters):
                        comm.allreduce_grads(table, "fp32")
                    b.record(stream)
                    torch.cuda.synchronize()
                    eager_us = a.elapsed_time(b) / args.iters * 1e3
                    # the same call captured once into a CUDA graph and
                    # replayed: no host submission cost between calls, so
                    # small sizes show the device-side floor
                    graph = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(graph):
                        comm.allreduce_grads(table, "fp32")
                    for _ in range(3):
                        graph.replay()
                    torch.cuda.synchronize()
                    a.record(stream)
                    for _ in range(args.iters):
                        graph.replay()
                    b.record(stream)
                    torch.cuda.synchronize()
                    comm.poll_error()
                    print(json.dumps({"what": "emulated pack + all-reduce per call (barriers live), flat fp32",
                                      "N": N, "bytes": S, "algo": algo, "us_per_call": eager_us,
                                      "us_per_call_graph": a.elapsed_time(b) / args.iters * 1e3}),
                          flush=True)
                    del graph
                finally:
                    comm.finalize()
            del g
    torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
