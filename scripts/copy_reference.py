#!/usr/bin/env python
"""Size-matched copy references for the pack kernel (a1): torch's own
device copy of the ResNet-50 gradient bytes (fp32 -> fp32, 8 B/param) and
cast copy (fp32 -> fp16, 6 B/param), CUDA events over 200 back-to-back
launches -- the same traffic shape as k_pack, so its ratio to these is the
kernel's efficiency at this size (launch ramp and tail included)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, iters=200):
    for _ in range(10):
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
    P = 25557032
    src = torch.randn(P, device="cuda")
    dst32 = torch.empty_like(src)
    dst16 = torch.empty(P, dtype=torch.float16, device="cuda")
    big = torch.randn(1 << 28, device="cuda")
    bigd = torch.empty_like(big)
    out = {
        "torch_copy_fp32_us": timed(lambda: dst32.copy_(src)),
        "torch_cast_fp16_us": timed(lambda: dst16.copy_(src)),
        "torch_copy_1GiB_gbs": 2 * big.numel() * 4 / (timed(lambda: bigd.copy_(big), 50) * 1e-6) / 1e9,
        "bytes_fp32": 8 * P, "bytes_fp16": 6 * P,
    }
    out["torch_copy_fp32_gbs"] = out["bytes_fp32"] / (out["torch_copy_fp32_us"] * 1e-6) / 1e9
    out["torch_cast_fp16_gbs"] = out["bytes_fp16"] / (out["torch_cast_fp16_us"] * 1e-6) / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
