#!/usr/bin/env python
"""Per-kernel timings of the step's kernels on ONE GPU (simulated-N mode):
pack (a1), all-reduce (a2, local HBM stands in for NVLink), update (a3), and
the fused N = 1 step -- each against its HBM roofline (algorithmic bytes /
CUDA-event time vs MEASURED_PEAKS.json hbm_gbs).  Prints one JSON line per
measurement; used to fill profiles/ and DESIGN.md §6.

    python scripts/kernel_bench.py [--iters 50]
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


def timed(fn, iters, stream):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(iters):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters * 1e3   # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--emulated", action="store_true",
                    help="N > 1 in the emulated world (cmn_init_emulated: the one-/two-shot, fused "
                         "and sharded barrier kernels as cooperative launches, barriers live)")
    args = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    shapes = synth.resnet50_shapes()
    sizes = [synth.numel(s) for s in shapes]
    P = sum(sizes)
    dev = "cuda:0"
    stream = torch.cuda.current_stream()
    params0 = synth.params(shapes)
    for N in [int(x) for x in args.worlds.split(",")]:
        g_host = synth.grads(shapes, workers=N)
        g = [[torch.from_numpy(x).to(dev) for x in gw] for gw in g_host]
        for dtype in ("fp32", "fp16"):
            c = 4 if dtype == "fp32" else 2
            for algo in (("oneshot", "twoshot") if N > 1 else ("identity",)):
                comm = ((Comm.emulated_world(N) if args.emulated else Comm.simulated_world(N))
                        if N > 1 else Comm.init(0, 1, 0))
                w = [torch.from_numpy(p.copy()).to(dev) for p in params0]
                comm.register_params(w)
                if N > 1:
                    comm.set_algo(algo)
                _, L = comm.layout()
                gg = comm.prepare(g if N > 1 else g[0])

                def ar():
                    comm.allreduce_grads(gg, dtype)

                def upd():
                    comm.allreduce_grads(gg, dtype)
                    comm.update_momentum_sgd(0.1, 0.9)

                t_ar = timed(ar, args.iters, stream)
                t_both = timed(upd, args.iters, stream)
                t_upd = t_both - t_ar
                rec = {"N": N, "dtype": dtype, "algo": algo,
                       "allreduce_incl_pack_us": t_ar, "update_us": t_upd,
                       "update_gbs": (16 + c) * P / (t_upd * 1e-6) / 1e9,
                       "update_frac": (16 + c) * P / (t_upd * 1e-6) / 1e9 / peak}
                if N == 1:
                    rec["pack_gbs"] = (4 + c) * P / (t_ar * 1e-6) / 1e9
                    rec["pack_frac"] = rec["pack_gbs"] / peak

                    def step():
                        comm.step(gg, dtype, 0.1, 0.9)
                    t_step = timed(step, args.iters, stream)
                    import time as _t
                    torch.cuda.synchronize()
                    h0 = _t.perf_counter()
                    for _ in range(args.iters):
                        comm.step(gg, dtype, 0.1, 0.9)
                    h1 = _t.perf_counter()
                    torch.cuda.synchronize()
                    rec["host_us_per_step_call"] = (h1 - h0) / args.iters * 1e6
                    # same step captured once into a CUDA graph and replayed
                    gr = torch.cuda.CUDAGraph()
                    s2 = torch.cuda.Stream()
                    s2.wait_stream(stream)
                    with torch.cuda.stream(s2):
                        comm.step(gg, dtype, 0.1, 0.9, s2)
                    torch.cuda.synchronize()
                    with torch.cuda.graph(gr):
                        comm.step(gg, dtype, 0.1, 0.9)
                    t_graph = timed(gr.replay, args.iters, stream)
                    rec["graph_step_us"] = t_graph
                    # NEXT-3 NVLS at one rank: pack + multimem.ld_reduce/st through the
                    # NVSwitch (2 S per direction over NVLink: ld_reduce fetch+return,
                    # st send+write-back)
                    try:
                        comm.set_algo("nvls")
                        t_nv = timed(ar, args.iters, stream)
                        rec["nvls_allreduce_incl_pack_us"] = t_nv
                        t_nv_only = t_nv - t_ar
                        rec["nvls_kernel_us_est"] = t_nv_only
                        rec["nvls_nvlink_gbs_per_direction"] = 2 * c * P / (t_nv_only * 1e-6) / 1e9
                    except Exception as e:  # noqa: BLE001 -- reported, not fatal
                        rec["nvls_error"] = str(e)
                    # NEXT-1: fused bias-corrected Adam from the packed buffer
                    # (28 B/param fp32 r, 26 B/param fp16 r: read r, w, m, v;
                    # write w, m, v)
                    comm.set_algo("auto")

                    def adam():
                        comm.allreduce_grads(gg, dtype)
                        comm.update_adam(1e-3, 0.9, 0.999, 1e-8, 1)
                    t_adam = timed(adam, args.iters, stream) - t_ar
                    rec["adam_update_us"] = t_adam
                    # the whole N = 1 Adam step straight from the gradients
                    # (28 B/param: read g, w, m, v; write w, m, v)
                    t_adam_step = timed(lambda: comm.step_adam(gg, dtype, 1e-3, 0.9, 0.999, 1e-8, 1),
                                        args.iters, stream)
                    rec["adam_step_us"] = t_adam_step
                    rec["adam_step_gbs"] = 28 * P / (t_adam_step * 1e-6) / 1e9
                    rec["adam_step_frac"] = rec["adam_step_gbs"] / peak
                    rec["adam_update_gbs"] = (24 + c) * P / (t_adam * 1e-6) / 1e9
                    rec["adam_update_frac"] = rec["adam_update_gbs"] / peak
                    rec["fused_step_us"] = t_step
                    rec["fused_step_gbs"] = 20 * P / (t_step * 1e-6) / 1e9
                    rec["fused_step_frac"] = rec["fused_step_gbs"] / peak
                else:
                    # simulated: N packs + N (oneshot) or 2N (twoshot) launches, all local HBM
                    rec["sim_note"] = "all N ranks' kernels on one GPU; local HBM stands in for NVLink"
                    rec["world"] = "emulated (barriers live)" if args.emulated else "simulated (barriers off)"
                    if algo == "twoshot":
                        # whole-step schedules: in simulation every rank's pack and
                        # all-reduce kernels run on this one GPU from local HBM, while
                        # the simulated ranks' shared parameter replica is updated once
                        # -- mechanics and local-memory cost, not an N-GPU time
                        sched = {}
                        for name, fused, pieces in (("serial", 0, 0), ("pipelined4", 0, 4),
                                                    ("fused", 1, 0), ("fused_push", 2, 0)):
                            comm.set_fused_update(fused)
                            comm.set_pipeline(pieces)
                            sched[name] = timed(lambda: comm.step(gg, dtype, 0.1, 0.9), args.iters, stream)
                        comm.set_fused_update(0)
                        sched["sharded"] = timed(lambda: comm.step_sharded(gg, dtype, 0.1, 0.9),
                                                 args.iters, stream)
                        rec["sim_step_us"] = sched
                print(json.dumps(rec), flush=True)
                comm.finalize()
                del w
        del g
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
