#!/usr/bin/env python
"""BASELINE config 1 (tiny MLP 784-100-100-10, 89,610 params): a latency
config -- its rooflines (0.2 us of HBM traffic at N = 1, 0.4 us of NVLink at
N = 2) sit far below launch latency, so report what a step costs instead:
device time per step (CUDA events around back-to-back steps), host time per
API call, and the same step replayed from a captured CUDA graph.

    python scripts/latency_bench.py [--iters 500]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1908_00213_b200 import Comm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=500)
    a = ap.parse_args()
    shapes = synth.mlp_shapes()
    stream = torch.cuda.Stream()
    for N, mode in ((1, "cmn_init"), (2, "simulated"), (8, "simulated")):
        for dtype in ("fp32", "fp16"):
            comm = Comm.init(0, 1, 0) if N == 1 else Comm.simulated_world(N)
            w = [torch.from_numpy(p).cuda() for p in synth.params(shapes)]
            comm.register_params(w)
            g = synth.grads(shapes, workers=N)
            gt = comm.prepare([torch.from_numpy(x).cuda() for x in g[0]] if N == 1 else
                              [[torch.from_numpy(x).cuda() for x in gw] for gw in g])
            rec = {"config": "BASELINE config 1 (MLP 784-100-100-10)", "N": N, "comm": mode,
                   "dtype": dtype, "params": int(sum(x.numel() for x in w))}
            with torch.cuda.stream(stream):
                for _ in range(20):
                    comm.step(gt, dtype, 0.1, 0.9, stream)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                h0 = time.perf_counter()
                e0.record(stream)
                for _ in range(a.iters):
                    comm.step(gt, dtype, 0.1, 0.9, stream)
                e1.record(stream)
                h1 = time.perf_counter()
                torch.cuda.synchronize()
                rec["device_us_per_step"] = e0.elapsed_time(e1) / a.iters * 1e3
                rec["host_us_per_call"] = (h1 - h0) / a.iters * 1e6
                rec["launches_per_step"] = None
                before = comm.kernel_launches
                comm.step(gt, dtype, 0.1, 0.9, stream)
                rec["launches_per_step"] = comm.kernel_launches - before
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph, stream=stream):
                    comm.step(gt, dtype, 0.1, 0.9, stream)
                graph.replay()
                torch.cuda.synchronize()
                e0.record(stream)
                for _ in range(a.iters):
                    graph.replay()
                e1.record(stream)
                torch.cuda.synchronize()
                rec["graph_replay_us_per_step"] = e0.elapsed_time(e1) / a.iters * 1e3
            print(json.dumps(rec), flush=True)
            comm.finalize()


if __name__ == "__main__":
    main()
