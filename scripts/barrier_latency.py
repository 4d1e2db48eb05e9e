#!/usr/bin/env python
"""Latency of the cross-rank barrier kernels on one GPU: small all-reduces in
the emulated world (cmn_init_emulated: every rank in ONE cooperative launch,
barriers live) next to the simulated world (the same kernels, barriers off,
one launch per rank).  Each measurement is a CUDA graph of `--calls`
back-to-back cmn_allreduce_grads calls replayed `--reps` times, so no host
submission cost enters; the figure is device µs per call (all ranks' packs +
the all-reduce).  Used to A/B the barrier's memory-ordering variant
(build switch CMN_BARRIER_VARIANT, cmn_device.cuh).

    python scripts/barrier_latency.py [--worlds 2,8] [--elems 256,16384,262144]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1908_00213_b200 import Comm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--worlds", default="2,8")
    ap.add_argument("--elems", default="256,16384,262144")
    ap.add_argument("--calls", type=int, default=20)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--variant", default=os.environ.get("CMN_EXTRA_NVFLAGS", "default"))
    ap.add_argument("--ctas", default="0", help="collective CTAs per rank to try (0 = library default)")
    ap.add_argument("--kinds", default="emulated,simulated")
    args = ap.parse_args()
    dev = "cuda:0"
    stream = torch.cuda.current_stream()
    for N in [int(x) for x in args.worlds.split(",")]:
        for n in [int(x) for x in args.elems.split(",")]:
            g = [torch.empty(n, device=dev).uniform_(-1e-2, 1e-2) for _ in range(N)]
            for kind in args.kinds.split(","):
                for ctas in [int(x) for x in args.ctas.split(",")]:
                    for algo in ("oneshot", "twoshot"):
                        comm = Comm.emulated_world(N) if kind == "emulated" else Comm.simulated_world(N)
                        try:
                            w = torch.zeros(n, device=dev)
                            comm.register_params([w])
                            comm.set_algo(algo)
                            comm.set_ctas(ctas, 0)
                            table = comm.prepare(g)
                            for _ in range(3):
                                comm.allreduce_grads(table, "fp32")
                            torch.cuda.synchronize()
                            graph = torch.cuda.CUDAGraph()
                            with torch.cuda.graph(graph):
                                for _ in range(args.calls):
                                    comm.allreduce_grads(table, "fp32")
                            for _ in range(2):
                                graph.replay()
                            torch.cuda.synchronize()
                            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                            a.record(stream)
                            for _ in range(args.reps):
                                graph.replay()
                            b.record(stream)
                            torch.cuda.synchronize()
                            comm.poll_error()
                            us = a.elapsed_time(b) / (args.reps * args.calls) * 1e3
                            print(json.dumps({"variant": args.variant, "kind": kind, "N": N, "elems": n,
                                              "algo": algo, "ctas": ctas, "us_per_call": us}), flush=True)
                            del graph
                        finally:
                            comm.finalize()
            del g


if __name__ == "__main__":
    main()
