#!/usr/bin/env python
"""Small fixed workload for ncu captures (one GPU): R50 gradient set,
`--mode n1` runs pack (allreduce_grads at N=1) + update + the fused step;
`--mode sim8` runs simulated-N=8 two-shot/one-shot all-reduce + update."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1908_00213_b200 import Comm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="n1", choices=["n1", "sim8", "adam", "adam_step", "fused8", "push8", "sharded8"])
    ap.add_argument("--dtype", default="fp32")
    ap.add_argument("--algo", default="twoshot")
    ap.add_argument("--iters", type=int, default=3)
    a = ap.parse_args()
    shapes = synth.resnet50_shapes()
    N = 8 if a.mode.endswith("8") else 1
    comm = Comm.init(0, 1, 0) if N == 1 else Comm.simulated_world(N)
    w = [torch.from_numpy(p).cuda() for p in synth.params(shapes)]
    comm.register_params(w)
    if N > 1:
        comm.set_algo(a.algo)
        comm.set_pipeline(0)
    g = synth.grads(shapes, workers=N)
    gt = comm.prepare([[torch.from_numpy(x).cuda() for x in gw] for gw in g] if N > 1
                      else [torch.from_numpy(x).cuda() for x in g[0]])
    if a.mode in ("fused8", "push8"):
        comm.set_fused_update(2 if a.mode == "push8" else 1)
    for _ in range(a.iters if a.mode in ("fused8", "push8", "sharded8") else 0):
        if a.mode in ("fused8", "push8"):
            comm.step(gt, a.dtype, 0.1, 0.9)
        else:
            comm.step_sharded(gt, a.dtype, 0.1, 0.9)
    for _ in range(a.iters if a.mode in ("n1", "sim8") else 0):
        comm.allreduce_grads(gt, a.dtype)
        comm.update_momentum_sgd(0.1, 0.9)
        if N == 1:
            comm.step(gt, a.dtype, 0.1, 0.9)
    for k in range(a.iters if a.mode == "adam_step" else 0):
        comm.step_adam(gt, a.dtype, 1e-3, 0.9, 0.999, 1e-8, k + 1)
    for k in range(a.iters if a.mode == "adam" else 0):
        comm.allreduce_grads(gt, a.dtype)
        comm.update_adam(1e-3, 0.9, 0.999, 1e-8, k + 1)
    torch.cuda.synchronize()
    comm.finalize()


if __name__ == "__main__":
    main()
