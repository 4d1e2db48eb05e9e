#!/usr/bin/env python
"""Piece-plan A/B for the N = 1 host-buffer step (cmn_step_host_packed).

    python scripts/e2e_plan_probe.py [--rounds 5]

Each plan is a CMN_E2E_WEIGHTS string (relative piece sizes in layout order;
"" = the library default kE2EWeights).  Plans are timed in interleaved rounds
(CUDA events around 10 back-to-back calls, the bench's e2e protocol) so box
drift hits every plan alike; medians are printed as one JSON line per plan,
after bare H2D / D2H / bidirectional copies of the same bytes for reference.
The result is checked bitwise against the default plan (plans only move
piece boundaries)."""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_1908_00213_b200 import Comm  # noqa: E402

PLANS = {
    "default(1,2,4,8x6,4,2,1)": "",
    "default, per-tensor D2H": "per_tensor",
    "7:1,4,16,16,16,4,1": "1,4,16,16,16,4,1",
    "8:1,2,8,16,16,8,2,1": "1,2,8,16,16,8,2,1",
    "6:1,8,24,24,8,1": "1,8,24,24,8,1",
    "9:1,3,9,16,16,16,9,3,1": "1,3,9,16,16,16,9,3,1",
    "16:1,2,4,8x10,4,2,1": "1,2,4," + ",".join(["8"] * 10) + ",4,2,1",
    "5:1,16,32,16,1": "1,16,32,16,1",
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=5)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    shapes = synth.resnet50_shapes()
    g_np = synth.grads(shapes, workers=1)[0]
    w_np = synth.params(shapes)
    comm = Comm.init(0, 1, 0)
    try:
        w = [torch.from_numpy(x.copy()).to(dev) for x in w_np]
        comm.register_params(w)
        off, L = comm.layout()
        hg = torch.zeros(L, dtype=torch.float32).pin_memory()
        hw = torch.empty(L, dtype=torch.float32).pin_memory()
        for t, x in enumerate(g_np):
            hg[off[t]: off[t] + x.size].copy_(torch.from_numpy(x.reshape(-1)))
        stream = torch.cuda.current_stream()

        def set_plan(plan):
            os.environ["CMN_E2E_PER_TENSOR_D2H"] = "1" if plan == "per_tensor" else "0"
            os.environ["CMN_E2E_WEIGHTS"] = "" if plan == "per_tensor" else plan

        def run(plan, k=10):
            set_plan(plan)
            comm.step_host_packed(hg, hw, "fp32", 0.1, 0.9, stream)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(k):
                comm.step_host_packed(hg, hw, "fp32", 0.1, 0.9, stream)
            e1.record(stream)
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / k * 1e3

        # bitwise: one step from identical state under each plan
        ref = None
        for name, plan in PLANS.items():
            for t, x in enumerate(w_np):
                w[t].copy_(torch.from_numpy(x))
            comm.register_params(w)  # resets momentum
            set_plan(plan)
            comm.step_host_packed(hg, hw, "fp32", 0.1, 0.9, stream)
            torch.cuda.synchronize()
            out = hw.clone()
            if ref is None:
                ref = out
            assert torch.equal(out.view(torch.int32), ref.view(torch.int32)), name

        d = torch.empty(L, dtype=torch.float32, device=dev)
        s2 = torch.cuda.Stream()

        def copy_us(fn, k=5):
            fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(k):
                fn()
            e1.record(stream)
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / k * 1e3

        def both():
            s2.wait_stream(stream)
            d.copy_(hg, non_blocking=True)
            with torch.cuda.stream(s2):
                hw.copy_(d, non_blocking=True)
            stream.wait_stream(s2)
        print(json.dumps({"bare_h2d_us": copy_us(lambda: d.copy_(hg, non_blocking=True)),
                          "bare_d2h_us": copy_us(lambda: hw.copy_(d, non_blocking=True)),
                          "bare_both_us": copy_us(both)}), flush=True)
        times = {n: [] for n in PLANS}
        for _ in range(a.rounds):
            for n, plan in PLANS.items():
                times[n].append(run(plan))
        for n, ts in times.items():
            print(json.dumps({"plan": n, "weights": PLANS[n] if PLANS[n] not in ("", "per_tensor") else "kE2EWeights",
                              "params": "separate tensors (one per layer)", "e2e_us_median": statistics.median(ts),
                              "e2e_us": ts, "bitwise_equal_default": True}), flush=True)
    finally:
        os.environ.pop("CMN_E2E_WEIGHTS", None)
        os.environ.pop("CMN_E2E_PER_TENSOR_D2H", None)
        comm.finalize()


if __name__ == "__main__":
    main()
