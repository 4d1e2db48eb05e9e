#!/usr/bin/env python
"""NEXT-2 measurement: a real autograd ResNet-50 training step at N = 1 with
the update through multi_node_optimizer (optim.py -> libcmn) against the
same step with torch.optim.SGD(momentum, fused=True).

    python scripts/train_step_bench.py [--batch 32] [--steps 20] [--rounds 3]

torchvision ResNet-50 (random init, 161 parameter tensors in parameters()
order = synth.resnet50_shapes()), synthetic ImageNet-shaped batch (the
paper's 32 images per worker), fp32 compute (
TF32 tensor cores allowed for the convolutions, as torch's default cuDNN
setting), cross-entropy loss.  Arms, interleaved over --rounds rounds, CUDA
events around --steps whole steps (forward, backward, update):
  torch_sgd_fused      torch.optim.SGD(lr, momentum, fused=True)
  cmn                  MultiNodeOptimizer (cmn_step: k_update_direct)
  cmn_bucketed_8MB     MultiNodeOptimizer with bucket_bytes = 8 MB (backward
                       hooks launch the per-bucket exchange while backward runs)
Also times the update alone (the optimizer call after a finished backward)
for each arm.  Prints one JSON line per arm."""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1908_00213_b200 import Comm  # noqa: E402
from paper_1908_00213_b200.optim import create_multi_node_optimizer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--rounds", type=int, default=3)
    a = ap.parse_args()
    import torchvision
    dev = torch.device("cuda:0")
    torch.manual_seed(0)
    x = torch.randn(a.batch, 3, 224, 224, device=dev)
    y = torch.randint(0, 1000, (a.batch,), device=dev)
    lossf = torch.nn.CrossEntropyLoss()
    comms = []
    arms = {}
    for name in ("torch_sgd_fused", "cmn", "cmn_bucketed_8MB"):
        torch.manual_seed(1)
        model = torchvision.models.resnet50().to(dev)
        params = list(model.parameters())
        if name == "torch_sgd_fused":
            opt = torch.optim.SGD(params, lr=0.1, momentum=0.9, fused=True)
        else:
            comms.append(Comm.init(0, 1, 0))        # one communicator per model (one registration each)
            opt = create_multi_node_optimizer(params, comms[-1], lr=0.1, momentum=0.9,
                                              bucket_bytes=(8 << 20) if "bucketed" in name else None)
        arms[name] = (model, opt, len(params), sum(p.numel() for p in params))

    def one(model, opt):
        opt.zero_grad()
        lossf(model(x), y).backward()
        opt.step()

    def timed(fn, k):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(k):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / k

    for model, opt, _, _ in arms.values():          # warm-up (cuDNN autotune, allocator)
        for _ in range(5):
            one(model, opt)
    step_ms = {n: [] for n in arms}
    upd_us = {n: [] for n in arms}
    for _ in range(a.rounds):
        for n, (model, opt, _, _) in arms.items():
            step_ms[n].append(timed(lambda: one(model, opt), a.steps))
            if "bucketed" not in n:                   # update alone, grads already present
                upd_us[n].append(timed(opt.step, a.steps) * 1e3)
    try:
        for n, (model, opt, T, P) in arms.items():
            print(json.dumps({"arm": n, "model": "torchvision resnet50 (random init)", "tensors": T,
                              "params": P, "batch": a.batch, "step_ms_median": statistics.median(step_ms[n]),
                              "step_ms": step_ms[n],
                              "update_only_us_median": statistics.median(upd_us[n]) if upd_us[n] else None,
                              "images_per_s": a.batch / statistics.median(step_ms[n]) * 1e3}), flush=True)
    finally:
        for c in comms:
            c.finalize()


if __name__ == "__main__":
    main()
