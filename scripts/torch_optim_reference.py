#!/usr/bin/env python
"""Library comparison for the N = 1 update step (rows a1'/a3 and NEXT-1):
PyTorch's own multi-tensor optimizers on the same 161 ResNet-50 tensors
(separate allocations, as a model's parameters are) against cmn_step /
cmn_step_adam at N = 1.

    python scripts/torch_optim_reference.py

Arms (CUDA events over back-to-back steps on one stream, after warm-up; the
working set, 511 MB for SGD and 716 MB for Adam, exceeds the 126 MB L2):
  torch.optim.SGD(momentum=0.9, foreach=True)   multi-tensor-apply kernels
  torch.optim.SGD(momentum=0.9, fused=True)     one fused kernel per dtype group
  torch.optim.Adam(foreach=True) / (fused=True)
  cmn_step (k_update_direct) / cmn_step_adam (k_adam_direct)
Algorithmic bytes are the same for every arm (20 B/param SGD: read g, w, v,
write w, v; 28 B/param Adam: read g, w, m, v, write w, m, v), so the GB/s
columns compare directly.  torch's rounding differs (mul + add instead of
one fma), so no bitwise check here; parity of the cmn arms is in tests/.
Prints one JSON line per arm."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_1908_00213_b200 import Comm  # noqa: E402


def timed(fn, iters=100, warm=20):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters * 1e3


def main():
    dev = torch.device("cuda:0")
    shapes = synth.resnet50_shapes()
    P = sum(synth.numel(s) for s in shapes)
    g_np = synth.grads(shapes, workers=1)[0]
    w_np = synth.params(shapes)
    out = []

    def report(arm, us, bpp):
        d = {"arm": arm, "us": us, "params": P, "tensors": len(shapes), "bytes_per_param": bpp,
             "gbs": bpp * P / (us * 1e-6) / 1e9}
        out.append(d)
        print(json.dumps(d), flush=True)

    for name, cls, kw, bpp in (
            ("torch SGD foreach", torch.optim.SGD, dict(lr=0.1, momentum=0.9, foreach=True), 20),
            ("torch SGD fused", torch.optim.SGD, dict(lr=0.1, momentum=0.9, fused=True), 20),
            ("torch Adam foreach", torch.optim.Adam, dict(lr=1e-3, foreach=True), 28),
            ("torch Adam fused", torch.optim.Adam, dict(lr=1e-3, fused=True), 28)):
        ps = [torch.nn.Parameter(torch.from_numpy(x.copy()).to(dev)) for x in w_np]
        for p, g in zip(ps, g_np):
            p.grad = torch.from_numpy(g.copy()).to(dev)
        try:
            opt = cls(ps, **kw)
        except (RuntimeError, TypeError, ValueError) as e:  # option absent in this torch
            print(json.dumps({"arm": name, "unavailable": str(e)[:200]}), flush=True)
            continue
        report(name, timed(opt.step), bpp)
        del opt, ps
        torch.cuda.empty_cache()

    comm = Comm.init(0, 1, 0)
    try:
        w = [torch.from_numpy(x.copy()).to(dev) for x in w_np]
        g = [torch.from_numpy(x.copy()).to(dev) for x in g_np]
        comm.register_params(w)
        table = comm.prepare(g)
        report("cmn_step (k_update_direct)", timed(lambda: comm.step(table, "fp32", 0.1, 0.9)), 20)
        t = [0]

        def adam():
            t[0] += 1
            comm.step_adam(table, "fp32", 1e-3, 0.9, 0.999, 1e-8, t[0])
        report("cmn_step_adam (k_adam_direct)", timed(adam), 28)
    finally:
        comm.finalize()


if __name__ == "__main__":
    main()
