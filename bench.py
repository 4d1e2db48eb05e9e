#!/usr/bin/env python
"""Benchmark of the ChainerMN data-parallel update step (arXiv 1908.00213 §6)
on B200: BASELINE.json metric "allreduce+update step us and bus GB/s
(ResNet-50 grads) at 1/2/4/8 B200 vs roofline".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--dtype fp32|fp16]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1)
    python bench.py --impl reference ...                     (the CPU oracle arm)

A step is one pass of the whole hot path over the ResNet-50 gradient set
(161 tensors, 25,557,032 fp32 params): pack (+cast) -> all-reduce -> average +
momentum-SGD, through the C ABI (cmn_step).  At N = 1 the all-reduce is the
identity and cmn_step runs the fused direct kernel (no pack).  Inputs are
seeded synthetic gradients/params (synth/), resident in HBM before the timed
region; per-step traffic (511 MB) is 4x the L2, steps run back to back.  Rank 0 prints
ONE JSON line.
"""
from __future__ import annotations

import argparse
import contextlib
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "allreduce+update step µs and bus GB/s (ResNet-50 grads) at 1/2/4/8 B200 vs roofline"
FALLBACK_HBM_GBS = 6650.0

# N > 1 step schedules: name -> (fused-update mode: 0 off, 1 pull RS, 2 push
# pack+RS; pipeline pieces; all-reduce CTAs per SM; update CTAs per SM;
# 0 = library default).
SCHEDULES = {
    "pipelined2": (0, 2, 0, 0),
    "pipelined4": (0, 4, 0, 0),
    "pipelined8": (0, 8, 0, 0),
    "pipelined4_2cta": (0, 4, 2, 0),
    "fused": (1, 0, 0, 0),
    "fused_2cta": (1, 0, 2, 2),
    "fused_push": (2, 0, 0, 0),
    "fused_push_2cta": (2, 0, 2, 2),
    # one CTA per SM for every barrier kernel: a system-scope fence costs
    # more once two CTAs fence on one SM (emulated world)
    "fused_1cta": (1, 0, 1, 1),
    "fused_push_1cta": (2, 0, 1, 1),
    "serial": (0, 0, 0, 0),
    "serial_2cta": (0, 0, 2, 0),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)  # SURVEY d.1: 100 timed
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="cmn", choices=["cmn", "reference"])
    ap.add_argument("--dtype", default="fp32", choices=["fp32", "fp16"])
    ap.add_argument("--algo", default="auto", choices=["auto", "oneshot", "twoshot", "nccl", "nvls"])
    ap.add_argument("--schedule", default="auto",
                    choices=["auto"] + list(SCHEDULES),
                    help="N > 1 step schedule; auto = short max-over-ranks trial of each, fastest wins")
    ap.add_argument("--min-warmup-s", type=float, default=1.0,
                    help="keep warming up (untimed) at least this long so the clock sampler sees load")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=10.0,
                    help="cpu_baseline: time full-workload oracle steps for about this long (>= 3 steps)")
    ap.add_argument("--nvls", action="store_true",
                    help="N > 1: run the NVLS (multimem) all-reduce in THIS process right away (comparison, "
                         "and a headline candidate if it passes the runtime tolerance gate), skipping the "
                         "isolated probe below")
    ap.add_argument("--no-nvls-probe", action="store_true",
                    help="N > 1: skip the NVLS probe.  By default every rank first runs the NVLS all-reduce "
                         "in a CHILD process (its own process group and CUDA context), so a fault in the "
                         "never-before-executed multimem kernel cannot poison this run; only if every "
                         "rank's child passed the tolerance gate does this process set NVLS up itself "
                         "(comparison + headline candidate)")
    ap.add_argument("--nvls-child", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--sweep-budget-s", type=float, default=20.0,
                    help="N > 1: BASELINE config 5 -- packed-buffer sweep 64 KB .. 1 GB (fp32), the "
                         "hand-written all-reduce vs NCCL, bus GB/s; stops when this budget is spent "
                         "(0 = off)")
    ap.add_argument("--tune-budget-s", type=float, default=30.0,
                    help="N > 1 schedule autotune: stop trying candidates after this long "
                         "(candidates in a fixed order, the default schedule first)")
    return ap.parse_args()


# ----------------------------------------------------------------- helpers

@contextlib.contextmanager
def stdout_to_stderr():
    """Route fd 1 to stderr (native libraries, e.g. NCCL's version banner,
    must not add lines to the one-JSON-line stdout)."""
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    try:
        yield
    finally:
        sys.stdout.flush()
        os.dup2(saved, 1)
        os.close(saved)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, STREAM-style copy)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic(key: str):
    """dram bytes per launch of the dominant kernel from the committed ncu
    --set full summary (profiles/), or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    v = d.get(key)
    return None if v is None else float(v)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled while the GPU is loaded."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, ValueError):
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), line.strip()))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.t:
            self.t.join(timeout=2)

    def summary(self, t0: float, t1: float):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ts, line in self.rows:
            if not (t0 <= ts <= t1):
                continue
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def workload():
    import synth
    shapes = synth.resnet50_shapes()
    return shapes, [synth.numel(s) for s in shapes]


def workload_name(P: int, dtype: str, world: int) -> str:
    """config.workload, identical for both arms."""
    head = f"ResNet-50 gradient set (161 tensors, {P:,} fp32 params), {dtype} payload, "
    cfg = "BASELINE config 2" if dtype == "fp32" else "BASELINE config 3's fp16 payload"
    if world == 1:
        return (head + "data-parallel update step at N=1: the all-reduce is the identity, so the "
                f"step is the fused average + momentum-SGD update straight from the gradients, no pack ({cfg})")
    return (head + f"pack(+cast) -> all-reduce over {world} GPUs -> average + momentum-SGD step ({cfg})")


def common_config(P: int, T: int, L: int, dtype: str, world: int) -> dict:
    """The `config` object, identical in both arms (the driver compares them);
    everything arm-specific goes under the line's `details`."""
    return {"workload": workload_name(P, dtype, world), "n_tensors": T, "n_params": P, "padded_len": L,
            "comm_dtype": dtype, "lr": 0.1, "mu": 0.9, "parallelism": f"dp{world}",
            "l2": "inputs larger than L2: 20 B/param = 511 MB streamed per step vs 126 MB L2 "
                  "(no flush between steps)"}


# ------------------------------------------------------ CPU oracle baseline

def _oracle_inputs(n_workers: int):
    """The full workload on the host: n_workers' ResNet-50 gradients, the
    parameters, zero momentum (seeded synth/, like the GPU arm)."""
    import numpy as np

    import synth
    shapes, sizes = workload()
    g = synth.grads(shapes, workers=n_workers)
    w = synth.params(shapes)
    v = [np.zeros_like(x) for x in w]
    return sum(sizes), g, w, v


def oracle_step_time(n_workers: int, dtype: str, budget_s: float = 0.0, steps: int = 0,
                     warmup: int = 0, threads: int = 1):
    """Time the CPU oracle as it stands (oracle/cmn_oracle.c orc_step:
    pack + tree reduce + average + momentum SGD) on the FULL workload:
    `warmup` untimed + `steps` timed steps, or (steps = 0) steps for about
    budget_s seconds, at least 3.  threads > 1 runs the same oracle under
    SURVEY §8(d) d.5 (ii)'s elementwise partition across host threads
    (oracle.step_threaded, bit-identical output).  Returns (mean us per
    step, total timed seconds, timed steps, sample description)."""
    import oracle
    P, g, w, v = _oracle_inputs(n_workers)
    if threads > 1:
        def one():
            oracle.step_threaded(g, w, v, 0.1, 0.9, dtype, threads=threads)
    else:
        def one():
            oracle.step(g, w, v, 0.1, 0.9, dtype)
    for _ in range(warmup):
        one()
    n = 0
    t0 = time.perf_counter()
    while (steps and n < steps) or (not steps and (time.perf_counter() - t0 < budget_s or n < 3)):
        one()
        n += 1
    total = time.perf_counter() - t0
    how = "1 thread" if threads <= 1 else f"{threads} threads, elementwise partition"
    desc = (f"oracle/cmn_oracle.c orc_step (pack+tree-reduce+average+momentum-SGD, {how}) on the full "
            f"workload: all 161 ResNet-50 tensors ({P:,} params), {n_workers} simulated worker(s), {dtype}, "
            f"mean of {n} timed full steps after {warmup} untimed")
    return total / n * 1e6, total, n, desc


def _cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    """--impl reference: the CPU oracle on the host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    n = max(1, args.gpus)
    us, total_s, k, desc = oracle_step_time(n, args.dtype, steps=args.steps, warmup=args.warmup)
    shapes, sizes = workload()
    import oracle
    L = oracle.layout(sizes)[1]
    cfg = common_config(sum(sizes), len(sizes), L, args.dtype, n)
    line = {"impl": "reference", "metric": METRIC, "value": us, "unit": "us", "n_gpus": n,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": us / 1e3,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded counter-hash, synth/)", "config": cfg,
            "details": {"timed_region_s": total_s, "workers": f"{n} worker(s) simulated on the host CPU"},
            "cpu_baseline": {"value": us, "unit": "us", "cores": 1, "kind": "oracle", "sample": desc,
                             "cpu": _cpu_model()},
            "e2e": {"value": us, "unit": "us", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def all_ranks_agree(flag: bool) -> bool:
    """Collective over the default (gloo) group: True only if every rank
    passes True (MIN over ranks).  Every decision that selects which
    collectives run next (autotune budget, sweep budget) goes through it, so
    ranks whose clocks disagree never issue different collectives."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([1.0 if flag else 0.0], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return t.item() == 1.0


# ------------------------------------------------ the resident workload

def resident_workload(comm, rank, dev):
    """The ResNet-50 parameters in one flat device allocation laid out like
    the packed layout (a flat-parameter model, so the e2e D2H is one copy),
    registered with `comm`, and this rank's worker gradients resident in HBM
    behind a pre-marshalled pointer table.  Returns a dict."""
    import torch

    import synth
    import paper_1908_00213_b200.cmn as cmn_mod
    shapes, sizes = workload()
    off, L, _ = cmn_mod.plan_layout(shapes)
    flat_w = torch.empty(L, dtype=torch.float32, device=dev)
    p0 = synth.params(shapes)
    w = []
    for t, s in enumerate(shapes):
        view = flat_w[off[t]: off[t] + sizes[t]].view(s)
        view.copy_(torch.from_numpy(p0[t]).view(s))
        w.append(view)
    comm.register_params(w)
    g_host = [synth.grad_tensor(n, t, worker=rank) for t, n in enumerate(sizes)]   # this rank's worker
    flat_g = torch.empty(L, dtype=torch.float32, device=dev)
    g = []
    for t, s in enumerate(shapes):
        view = flat_g[off[t]: off[t] + sizes[t]]
        view.copy_(torch.from_numpy(g_host[t]))
        g.append(view)
    return {"shapes": shapes, "sizes": sizes, "off": off, "L": L, "flat_w": flat_w, "w": w,
            "flat_g": flat_g, "g": comm.prepare(g), "g_host": g_host}


def timed_calls_us(fn, stream, n=10, warm=3, barrier=None):
    """Device µs per call of fn(): `warm` untimed calls, then n calls between
    CUDA events on `stream`; max over ranks when a process group exists."""
    import torch
    import torch.distributed as dist
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    if barrier:
        barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(n):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / n], dtype=torch.float64)
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()) * 1e3


def nvls_tolerance_ratio(comm, wl, dtype, stream, dev, world, algo="nvls"):
    """The NVLS sum (switch order) against the two-shot tree sum of the same
    gradients, elementwise within the north-star tolerance:
    |r_nvls - r_tree| <= 1e-5 * sum_i |g_i| (fp32 payload) or
    2e-3 * sum_i |g_i| + N * 2^-24 (fp16), with sum_i |g_i| itself
    all-reduced (two-shot) from each rank's |g|.  Max violation ratio over
    all elements and ranks; <= 1 passes.  Leaves `algo` selected."""
    import torch
    import torch.distributed as dist
    L, off, sizes, flat_g = wl["L"], wl["off"], wl["sizes"], wl["flat_g"]
    tdt = torch.float32 if dtype == "fp32" else torch.float16
    comm.set_algo("twoshot")
    comm.allreduce_grads(wl["g"], dtype, stream)
    r_tree = torch.empty(L, dtype=tdt, device=dev)
    comm.copy_reduced(comm.rank, r_tree, stream)
    comm.update_momentum_sgd(0.0, 0.0, stream)          # consume (state hygiene)
    abs_flat = flat_g.abs()
    abs_g = comm.prepare([abs_flat[off[t]: off[t] + sizes[t]] for t in range(len(sizes))])
    comm.allreduce_grads(abs_g, "fp32", stream)
    sum_abs = torch.empty(L, dtype=torch.float32, device=dev)
    comm.copy_reduced(comm.rank, sum_abs, stream)
    comm.update_momentum_sgd(0.0, 0.0, stream)
    comm.set_algo(algo)
    comm.allreduce_grads(wl["g"], dtype, stream)
    r_nv = torch.empty(L, dtype=tdt, device=dev)
    comm.copy_reduced(comm.rank, r_nv, stream)
    comm.update_momentum_sgd(0.0, 0.0, stream)
    torch.cuda.synchronize()
    diff = (r_nv.float() - r_tree.float()).abs()
    bound = (1e-5 * sum_abs if dtype == "fp32" else 2e-3 * sum_abs + world * 2.0 ** -24)
    ratio = torch.tensor([float((diff / bound.clamp_min(1e-30)).max())], dtype=torch.float64)
    if dist.is_initialized() and world > 1:
        dist.all_reduce(ratio, op=dist.ReduceOp.MAX)
    return float(ratio.item())


def replicas_digest_equal(flat_w, dev, world):
    """Bitwise replica consistency: a weighted
    digest of every rank's parameter bits, all-gathered and compared."""
    import torch
    import torch.distributed as dist
    bits = flat_w.view(torch.int32).to(torch.int64)
    wgt = torch.arange(bits.numel(), device=dev, dtype=torch.int64) % 1009 + 1
    digest = torch.stack([bits.sum(), (bits * wgt).sum()]).cpu()
    all_d = [torch.zeros_like(digest) for _ in range(world)]
    dist.all_gather(all_d, digest)
    return all(torch.equal(d, all_d[0]) for d in all_d)


# ----------------------------------------------- NVLS probe (N > 1 only)
#
# k_nvls (multimem.ld_reduce / multimem.st over a multicast object) has
# never executed: the one-GPU boxes this was developed on refuse multicast
# objects.  A fault in it would poison the CUDA context of the whole N > 1
# bench, so by default each rank first runs it in a child process of its own
# (own process group on another port, own CUDA context, 10 s barrier
# timeout); the bench adopts NVLS only when every rank's child came back
# with a passed tolerance gate.

def run_nvls_child(args):
    """bench.py --nvls-child (spawned by nvls_probe): set NVLS up, gate its
    sums against the tree, time it, print one JSON object."""
    import datetime

    import torch
    import torch.distributed as dist

    from paper_1908_00213_b200 import Comm
    from paper_1908_00213_b200.cmn import CmnError
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("gloo", init_method=os.environ["CMN_NVLS_CHILD_INIT"], rank=rank,
                            world_size=world, timeout=datetime.timedelta(seconds=90))
    algo = os.environ.get("CMN_TEST_NVLS_PROBE_ALGO", "nvls")    # tests: plumbing with a P2P algo
    out = {"probe": "child process (own process group and CUDA context)", "algo": algo}
    comm = Comm.init(rank, world, local, dist.group.WORLD)
    try:
        comm.set_timeout(10000)
        wl = resident_workload(comm, rank, dev)
        stream = torch.cuda.current_stream(dev)
        try:
            with stdout_to_stderr():
                comm.set_algo(algo)
            ok = all_ranks_agree(True)
        except CmnError as e:
            all_ranks_agree(False)
            out["unavailable"] = str(e)[:200]
            ok = False
        try:
            if ok and os.environ.get("CMN_TEST_NVLS_SETUP_ONLY") == "1":
                out["setup_only"] = True      # tests: stop before any barrier kernel runs
            elif ok:
                _nvls_child_measure(comm, wl, args, stream, dev, world, algo, out)
            comm.poll_error()
        except CmnError as e:
            out["error"] = str(e)[:200]
            out["passed"] = False
    finally:
        with stdout_to_stderr():
            comm.finalize()
    print(json.dumps(out))
    sys.stdout.flush()
    dist.destroy_process_group()
    return 0


def _nvls_child_measure(comm, wl, args, stream, dev, world, algo, out):
    """The child's gate and timings: the tolerance ratio against the tree
    sums, then (if it passes) pack + all-reduce alone and the serial and
    pipelined steps with this algorithm, and the replicas' bitwise equality."""
    import torch
    import torch.distributed as dist
    ratio = nvls_tolerance_ratio(comm, wl, args.dtype, stream, dev, world, algo)
    out["tolerance_ratio_vs_tree"] = ratio
    out["passed"] = ratio <= 1.0
    if ratio > 1.0:
        return
    S_bus = 2 * (world - 1) / world * (4 if args.dtype == "fp32" else 2) * sum(wl["sizes"])
    g = wl["g"]
    us = timed_calls_us(lambda: comm.allreduce_grads(g, args.dtype, stream), stream, barrier=dist.barrier)
    comm.update_momentum_sgd(0.1, 0.9, stream)          # consume (state hygiene)
    out["allreduce_incl_pack_us"] = us
    out["allreduce_incl_pack_bus_gbs"] = S_bus / (us * 1e-6) / 1e9
    for name, pieces in (("serial", 0), ("pipelined4", 4)):
        comm.set_pipeline(pieces)
        t = timed_calls_us(lambda: comm.step(g, args.dtype, 0.1, 0.9, stream), stream, barrier=dist.barrier)
        out[f"{name}_step_us"] = t
        out[f"{name}_step_bus_gbs"] = S_bus / (t * 1e-6) / 1e9
    torch.cuda.synchronize()
    out["replicas_bitwise_equal"] = replicas_digest_equal(wl["flat_w"], dev, world)


def nvls_probe(args, rank, world, local, timeout_s=300):
    """Run run_nvls_child on every rank at once (collective: every parent
    rank calls it).  Returns (this rank's child result dict, True if every
    rank's child passed with the real NVLS algorithm)."""
    import socket

    import torch.distributed as dist
    port = [0]
    if rank == 0:
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port[0] = s.getsockname()[1]
        s.close()
    dist.broadcast_object_list(port, src=0)
    addr = os.environ.get("MASTER_ADDR", "127.0.0.1")
    env = dict(os.environ, CMN_NVLS_CHILD_INIT=f"tcp://{addr}:{port[0]}",
               RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(local))
    cmd = [sys.executable, os.path.abspath(__file__), "--nvls-child", "--dtype", args.dtype,
           "--gpus", str(world)]
    t0 = time.time()
    try:
        p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=timeout_s)
        lines = [x for x in p.stdout.splitlines() if x.startswith("{")]
        if p.returncode == 0 and lines:
            res = json.loads(lines[-1])
        else:
            tail = (p.stderr or "").strip().splitlines()[-3:]
            res = {"probe": "child process", "unavailable": f"probe process exited {p.returncode}: "
                                                            + " | ".join(tail)[:300]}
    except subprocess.TimeoutExpired:
        res = {"probe": "child process", "unavailable": f"probe process timed out after {timeout_s} s"}
    res["probe_s"] = round(time.time() - t0, 1)
    passed = bool(res.get("passed")) and res.get("algo") == "nvls" and res.get("replicas_bitwise_equal")
    return res, all_ranks_agree(passed)


# ------------------------------------------------- config 5 (N > 1 only)

SWEEP_BYTES = [64 << 10, 1 << 20, 16 << 20, 256 << 20, 1 << 30]


def config5_sweep(args, rank, world, local, group, dev, stream):
    """BASELINE config 5 at this N: one flat fp32 "tensor" of S bytes, S from
    64 KB to 1 GB; pack + all-reduce alone (cmn_allreduce_grads, no update)
    with the hand-written kernels (algo auto: one-shot <= 1 MB, else
    two-shot) and with NCCL, 10 calls after 3 warm-up, max over ranks; bus
    GB/s = 2(N-1)/N S / t.  A separate communicator (one re-registration per
    size, a collective); the inputs are device-generated (timing only, no
    parity claim).  Stops when --sweep-budget-s is spent (decided
    collectively, so every rank runs the same sizes)."""
    import torch
    import torch.distributed as dist

    from paper_1908_00213_b200 import Comm
    from paper_1908_00213_b200.cmn import CmnError
    t0 = time.time()
    out = []
    c2 = Comm.init(rank, world, local, group)

    def time_ar(table):
        for _ in range(3):
            c2.allreduce_grads(table, "fp32", stream)
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(10):
            c2.allreduce_grads(table, "fp32", stream)
        b.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / 10 * 1e3], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        c2.update_momentum_sgd(0.0, 0.0, stream)      # consume (state hygiene)
        return float(t.item())

    nccl_ok = None
    try:
        for S in SWEEP_BYTES:
            if not all_ranks_agree(time.time() - t0 < args.sweep_budget_s):
                break
            n = S // 4
            w = torch.zeros(n, dtype=torch.float32, device=dev)
            gen = torch.Generator(device=dev).manual_seed(190800213 + rank)
            g = torch.empty(n, dtype=torch.float32, device=dev).uniform_(-1e-2, 1e-2, generator=gen)
            c2.register_params([w])
            c2.set_algo("auto")
            table = c2.prepare([g])
            bus = 2 * (world - 1) / world * S
            rec = {"bytes": S, "dtype": "fp32"}
            us = time_ar(table)
            rec.update(cmn_us=us, cmn_bus_gbs=bus / (us * 1e-6) / 1e9)
            if nccl_ok is False:
                rec["nccl"] = "unavailable (see the first size)"
            else:
                with stdout_to_stderr():
                    try:
                        c2.set_algo("nccl")
                        nccl_ok = True
                    except CmnError as e:
                        nccl_ok = False
                        rec["nccl"] = f"unavailable: {str(e)[:120]}"
                    if nccl_ok:
                        un = time_ar(table)
                        rec.update(nccl_us=un, nccl_bus_gbs=bus / (un * 1e-6) / 1e9)
            out.append(rec)
            del table, g, w
    finally:
        with stdout_to_stderr():
            c2.finalize()
    torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------- the bench

def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.nvls_child:
        return run_nvls_child(args)

    import torch
    import torch.distributed as dist

    from paper_1908_00213_b200 import Comm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        # NCCL (the measured comparison) reports its communicator (nranks,
        # NVLS / ring choice); every NCCL call below runs with fd 1 routed to
        # stderr, so those lines never reach the one-line stdout
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,ENV,TUNING")
    if args.gpus != world and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # one process per GPU.  Ranks whose kernels spin on each other's flags
    # are never time-sliced on one GPU (B200_PROFILING.md: nothing guarantees
    # they run together; 2 and 4 such processes on one B200 raised Xid 109)
    ndev = torch.cuda.device_count()
    if world > 1 and world > ndev:
        raise SystemExit(f"bench.py: {world} ranks need {world} GPUs, this box has {ndev} "
                         "(ranks are never time-sliced on one GPU)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        group = dist.group.WORLD

    comm = Comm.init(rank, world, local, group)
    wl = resident_workload(comm, rank, dev)      # registers the parameters
    shapes, sizes, off, L = wl["shapes"], wl["sizes"], wl["off"], wl["L"]
    flat_w, g, g_host = wl["flat_w"], wl["g"], wl["g_host"]
    P, T = sum(sizes), len(sizes)
    if args.algo != "auto" and world > 1:
        comm.set_algo(args.algo)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()

    nsm = torch.cuda.get_device_properties(dev).multi_processor_count

    def set_schedule(name, algo=None):
        if name.startswith("nvls"):     # in-switch all-reduce: "nvls" (serial), "nvls_<schedule>"
            algo, name = "nvls", name[5:] or "serial"
        if world > 1:
            comm.set_algo(algo or args.algo)
        fused, pieces, ar_x, upd_x = SCHEDULES[name]
        comm.set_fused_update(fused)
        comm.set_pipeline(pieces)
        comm.set_ctas(min(1024, ar_x * nsm), min(1024, upd_x * nsm))

    schedule, trials, comparisons = "identity (N=1 fused direct update)", None, {}
    if world > 1:
        # Runtime schedule choice: every rank times each candidate (max over
        # ranks, so all ranks pick the same one); switching schedules between
        # calls is safe (every buffer reuse is behind a start barrier).
        # fixed order, the library default (pipelined, 4 pieces) first: a
        # zero budget runs the default deterministically
        order = ["pipelined4"] + [n for n in SCHEDULES if n != "pipelined4"]
        cands = order if args.schedule == "auto" else [args.schedule]
        t_tune0 = time.time()

        def budget_left():
            """Collective: every rank gets the same answer (each rank's own
            clock decides, MIN over ranks), so all ranks try the same
            candidates -- a divergent choice would pair different
            collectives across ranks."""
            return all_ranks_agree(time.time() - t_tune0 < args.tune_budget_s)

        def trial_us():
            for _ in range(3):
                comm.step(g, args.dtype, 0.1, 0.9, stream)
            torch.cuda.synchronize()
            barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(10):
                comm.step(g, args.dtype, 0.1, 0.9, stream)
            b.record(stream)
            torch.cuda.synchronize()
            t = torch.tensor([a.elapsed_time(b) / 10], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item()) * 1e3

        def capture_step():
            """One step of the current schedule captured into a CUDA graph
            (graph-safe schedules only: their buffer reuse is barrier-ordered
            and barrier epochs live on the device, so replays stay paired
            across ranks); None if the schedule refuses capture."""
            from paper_1908_00213_b200.cmn import CmnError as _E
            comm.step(g, args.dtype, 0.1, 0.9, stream)          # internal streams exist
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            try:
                with torch.cuda.graph(graph):
                    comm.step(g, args.dtype, 0.1, 0.9)          # on the capture stream
            except _E:
                return None
            return graph

        def trial_graph_us(graph):
            for _ in range(3):
                graph.replay()
            torch.cuda.synchronize()
            barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(10):
                graph.replay()
            b.record(stream)
            torch.cuda.synchronize()
            t = torch.tensor([a.elapsed_time(b) / 10], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item()) * 1e3

        trials = {}
        for name in cands:
            set_schedule(name)
            trials[name] = trial_us()
            if not budget_left():        # collective: all ranks stop at the same candidate
                break
        # The same schedules replayed from a captured CUDA graph (no host
        # launch cost per step: the pipelined step is ~7 API calls per piece).
        for name in ("pipelined4", "pipelined8", "fused", "fused_push"):
            if args.schedule != "auto" or name not in trials:
                continue
            if not budget_left():
                break
            set_schedule(name)
            gr = capture_step()
            if gr is not None:
                trials[name + "_graph"] = trial_graph_us(gr)
            del gr
        # Comparisons: the same step with the all-reduce done by NCCL (the
        # north star's measured comparison, never a headline candidate) and
        # by the NVLS in-switch kernel (tolerance-only parity; a headline
        # candidate once its sums pass the tolerance gate against the tree
        # sums on this box).  Resource setup is collective and fails on
        # every rank alike.
        from paper_1908_00213_b200.cmn import CmnError
        S_bus = 2 * (world - 1) / world * (4 if args.dtype == "fp32" else 2) * P

        def allreduce_only_us():
            """pack(+cast) + all-reduce alone (cmn_allreduce_grads, no
            update), 10 calls, max over ranks: config 5's quantity at the
            R50 size, for the hand-written kernels and NCCL alike."""
            for _ in range(3):
                comm.allreduce_grads(g, args.dtype, stream)
            torch.cuda.synchronize()
            barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(10):
                comm.allreduce_grads(g, args.dtype, stream)
            b.record(stream)
            torch.cuda.synchronize()
            t = torch.tensor([a.elapsed_time(b) / 10], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            comm.update_momentum_sgd(0.1, 0.9, stream)      # consume (state hygiene)
            return float(t.item()) * 1e3

        set_schedule("serial", "auto")
        us_ar = allreduce_only_us()
        comparisons["cmn"] = {"allreduce_incl_pack_us": us_ar,
                              "allreduce_incl_pack_bus_gbs": S_bus / (us_ar * 1e-6) / 1e9}
        # NVLS: by default proven first in isolated child processes
        # (nvls_probe); this process sets it up only if every rank's child
        # passed the tolerance gate with bitwise-equal replicas.
        nvls_ok, probe = bool(args.nvls), None
        if not args.nvls and not args.no_nvls_probe:
            probe, nvls_ok = nvls_probe(args, rank, world, local)
        if not nvls_ok:
            why = ("probe skipped (--no-nvls-probe)" if probe is None else
                   probe.get("unavailable") or probe.get("error") or
                   "the isolated probe did not pass the tolerance gate on every rank")
            comparisons["nvls"] = {"unavailable": why, "probe": probe}
        for alt in ("nccl", "nvls") if nvls_ok else ("nccl",):
            with stdout_to_stderr():        # NCCL INFO lines -> stderr
                try:
                    comm.set_algo(alt)
                except CmnError as e:
                    comparisons[alt] = {"unavailable": str(e)[:160], "probe": probe}
                    continue
                comparisons[alt] = {"probe": probe} if alt == "nvls" else {}
                if alt == "nvls":
                    # the same gate in this process before anything is timed
                    ratio = nvls_tolerance_ratio(comm, wl, args.dtype, stream, dev, world)
                    comparisons[alt]["tolerance_ratio_vs_tree"] = ratio
                    if ratio > 1.0:
                        comparisons[alt]["unavailable"] = f"tolerance gate failed (ratio {ratio:.3g})"
                        continue
                set_schedule("serial", alt)
                us_alt = allreduce_only_us()
                comparisons[alt]["allreduce_incl_pack_us"] = us_alt
                comparisons[alt]["allreduce_incl_pack_bus_gbs"] = S_bus / (us_alt * 1e-6) / 1e9
                for sched in ("serial", "pipelined4"):
                    set_schedule(sched, alt)
                    t_alt = trial_us()
                    comparisons[alt][f"{sched}_step_us"] = t_alt
                    comparisons[alt][f"{sched}_step_bus_gbs"] = S_bus / (t_alt * 1e-6) / 1e9
            if alt == "nvls" and args.schedule == "auto":
                # passed the gate on this box: the in-switch all-reduce is a
                # headline candidate (the north star's tolerance, not the
                # tree's bit pattern -- reading R2)
                for name in ("nvls", "nvls_serial_2cta", "nvls_pipelined4", "nvls_pipelined4_2cta"):
                    set_schedule(name)
                    trials[name] = trial_us()
        schedule = min(trials, key=trials.get)
        set_schedule(schedule[:-len("_graph")] if schedule.endswith("_graph") else schedule)

    # what the timed region runs per step: the eager call, or the replay of
    # the chosen schedule's captured graph
    def eager_step():
        comm.step(g, args.dtype, 0.1, 0.9, stream)

    run_step = eager_step
    if schedule.endswith("_graph"):
        step_graph = capture_step()
        run_step = step_graph.replay
    launches_before = comm.kernel_launches
    eager_step()                       # kernels one step launches (graph replays launch the same)
    torch.cuda.synchronize()
    launches_per_step = comm.kernel_launches - launches_before

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    t_load0 = time.time()
    # warm-up (untimed): at least W steps and at least --min-warmup-s seconds
    t_w = time.time()
    n_w = 0
    while n_w < args.warmup or time.time() - t_w < args.min_warmup_s:
        run_step()
        n_w += 1
        if n_w % 64 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()

    # Timed region: K back-to-back steps.  Per-step traffic (20 B/param =
    # 511 MB at N = 1) is 4x the 126 MB L2, so steps stream from HBM; no L2
    # reuse across steps is possible (each step starts at the layout head,
    # the L2 holds the previous step's tail).
    e_start = torch.cuda.Event(enable_timing=True)
    e_stop = torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    e_start.record(stream)
    for k in range(args.steps):
        run_step()
    e_stop.record(stream)
    torch.cuda.synchronize()
    barrier()
    launches = launches_per_step * args.steps
    t_load1 = time.time()
    total_ms = e_start.elapsed_time(e_stop)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms = total_ms / args.steps
    us = ms * 1e3

    # The dominant kernel's own device time: a second pass of K steps with the
    # library bracketing each launch of it with CUDA events on the stream it
    # runs on (the all-reduce kernels run on an internal stream at N > 1).
    comm.set_kernel_timing(True)
    barrier()
    for k in range(args.steps):
        eager_step()                   # (launches inside a graph replay are not bracketed)
    torch.cuda.synchronize()
    k_ms, k_count = comm.kernel_timing()
    comm.set_kernel_timing(False)
    if world > 1:
        t = torch.tensor([k_ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        k_ms = float(t.item())
    kernel_ms_per_step = k_ms / args.steps
    kernel_launches_per_step = k_count / args.steps

    # Per-step distribution (median / mean / std over the
    # timed steps, max over ranks): a third pass with events between steps.
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    barrier()
    evs[0].record(stream)
    for k in range(args.steps):
        run_step()
        evs[k + 1].record(stream)
    torch.cuda.synchronize()
    per = [evs[k].elapsed_time(evs[k + 1]) * 1e3 for k in range(args.steps)]
    dstats = torch.tensor([statistics.median(per), statistics.fmean(per),
                           statistics.pstdev(per), min(per), max(per)], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(dstats, op=dist.ReduceOp.MAX)
    per_step = dict(zip(["median_us", "mean_us", "std_us", "min_us", "max_us"],
                        [float(x) for x in dstats]))
    per_step["n"] = args.steps

    # Transparency: the same step with a 256 MiB L2 write-flush before each
    # (untimed) -- the flush leaves up to 126 MB of dirty lines that the
    # step must write back, so this is a pessimistic "cold" figure.
    cold = []
    for k in range(min(args.steps, 20)):
        flush.add_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        run_step()
        b.record(stream)
        cold.append((a, b))
    torch.cuda.synchronize()
    cold_us = statistics.median(a.elapsed_time(b) for a, b in cold) * 1e3
    clocks = sampler.summary(t_load0, t_load1)
    sampler.stop()

    # Replica consistency: after the timed steps
    # every rank's parameters must be bitwise identical.
    replicas_equal = None
    if world > 1:
        replicas_equal = replicas_digest_equal(flat_w, dev, world)

    # ---- e2e: host buffers through cmn_step_host_packed (pinned H2D grads
    # in, updated params D2H out; pipelined over tensor ranges at N = 1)
    e2e = None
    if not args.no_e2e:
        hg_flat = torch.zeros(L, dtype=torch.float32).pin_memory()
        hw_flat = torch.empty(L, dtype=torch.float32).pin_memory()
        for t in range(T):
            hg_flat[off[t]: off[t] + sizes[t]].copy_(torch.from_numpy(g_host[t]))
        for _ in range(3):
            comm.step_host_packed(hg_flat, hw_flat, args.dtype, 0.1, 0.9, stream)
        torch.cuda.synchronize()
        barrier()
        ke = max(5, min(20, args.steps))
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(ke):
            comm.step_host_packed(hg_flat, hw_flat, args.dtype, 0.1, 0.9, stream)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        e_ms = e0.elapsed_time(e1) / ke
        if world > 1:
            t = torch.tensor([e_ms], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        # the PCIe bound of this e2e step: bare pinned H2D and D2H of the same
        # bytes, alone; with the call's H2D/update/D2H pipeline the floor is
        # about max(h2d, d2h), without overlap h2d + d2h
        dbuf = torch.empty(L, dtype=torch.float32, device=dev)

        def copy_us(fn):
            fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(5):
                fn()
            b.record(stream)
            torch.cuda.synchronize()
            return a.elapsed_time(b) / 5 * 1e3

        h2d_us = copy_us(lambda: dbuf.copy_(hg_flat, non_blocking=True))
        d2h_us = copy_us(lambda: hw_flat.copy_(dbuf, non_blocking=True))
        del dbuf
        e2e = {"value": e_ms * 1e3, "unit": "us", "h2d_bytes_per_step": 4 * L,
               "pcie_h2d_us": h2d_us, "pcie_d2h_us": d2h_us,
               "overlap_floor_us": max(h2d_us, d2h_us), "serial_floor_us": h2d_us + d2h_us,
               "d2h_bytes_per_step": 4 * L,
               "path": "cmn_step_host_packed: pinned host grads (packed layout) -> device, "
                       "step, params -> pinned host" + ("; pipelined over 12 ramped item ranges at N=1"
                                                         if world == 1 else
                                                         "; H2D/D2H per piece inside the pipelined "
                                                         "schedule" if schedule.startswith("pipelined")
                                                         else "; copies around the step")}

    with stdout_to_stderr():              # ncclCommDestroy may log
        comm.finalize()

    sweep = None
    if world > 1 and args.sweep_budget_s > 0:
        sweep = config5_sweep(args, rank, world, local, group, dev, stream)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel
    peak, peak_src = load_peaks()
    csz = 4 if args.dtype == "fp32" else 2
    timing_note = ("CUDA events around each launch on its own stream (cmn_set_kernel_timing), "
                   f"second pass of {args.steps} steps, max over ranks")
    if world == 1:
        kernel = "k_update_direct"
        alg_bytes = 20 * P              # read g, w, v; write w, v
        # The step is exactly one launch of this kernel on the caller's stream:
        # its average launch duration is the timed region / K (CUDA events
        # around the K back-to-back launches).  Bracketing every launch with
        # its own events (second pass) serialises launch tails and heads, so
        # that figure is reported beside it, not used.
        per_launch_ms = kernel_ms_per_step / max(kernel_launches_per_step, 1e-9)
        roof = {"bound": "hbm", "kernel": kernel,
                "achieved": alg_bytes / (ms * 1e-3) / 1e9,
                "peak": peak, "unit": "GB/s", "peak_source": peak_src,
                "algorithmic_bytes_per_launch": alg_bytes,
                "kernel_us_per_launch": ms * 1e3,
                "timing": f"CUDA events around the timed region of {args.steps} back-to-back "
                          "launches on the caller's stream (one launch per step)",
                "kernel_us_per_launch_isolated": per_launch_ms * 1e3,
                "isolated_timing": timing_note,
                "traffic": load_traffic(f"{kernel}_{args.dtype}")}
        roof["frac"] = roof["achieved"] / peak
        # context: the same achieved rate against the nominal HBM3e figure
        # (B200_PROFILING.md: 7.7 TB/s HGX) -- frac above 1 against the
        # measured 1:1 copy is possible because this kernel reads 3 streams
        # for every 2 it writes
        roof["nominal_peak"] = 7700.0
        roof["frac_of_nominal"] = roof["achieved"] / 7700.0
        # The conservative figure: per-step median with events between steps
        # (no overlap of one step's drain with the next one's launch)
        roof["achieved_per_step_median"] = alg_bytes / (per_step["median_us"] * 1e-6) / 1e9
        roof["frac_per_step_median"] = roof["achieved_per_step_median"] / peak
        bus = None
    else:
        S = csz * P
        bus_bytes = 2 * (world - 1) / world * S
        bus = bus_bytes / (ms * 1e-3) / 1e9
        kernel = ("k_pack_push + k_twoshot (local inbox reduce) + k_update_gather"
                  if schedule.startswith("fused_push")
                  else "k_twoshot (reduce-scatter) + k_update_gather" if schedule.startswith("fused")
                  else "k_nvls (multimem.ld_reduce / multimem.st)" if schedule.startswith("nvls")
                  else "k_oneshot / k_twoshot all-reduce")
        # The north-star quantity is the whole STEP against the bus roofline
        # (<= 248.5 us at N = 8 = 80 % of 900 GB/s): achieved =
        # bus bytes 2(N-1)/N S / ms_per_step, so exposed pack / update time
        # counts against it.  The collective kernels' own device time is
        # reported beside it (kernel_only).
        k_ach = bus_bytes / (kernel_ms_per_step * 1e-3) / 1e9
        roof = {"bound": "nvlink", "kernel": f"whole step, schedule {schedule}",
                "achieved": bus, "peak": 770.0, "unit": "GB/s",
                "peak_source": "measured peer copy 770 GB/s/direction (B200_PROFILING.md); "
                               "900 nominal in frac_of_nominal",
                "algorithmic_bytes_per_step": bus_bytes,
                "frac": bus / 770.0, "nominal_peak": 900.0, "frac_of_nominal": bus / 900.0,
                "timing": f"CUDA events around the timed region of {args.steps} steps, max over ranks",
                "kernel_only": {"kernel": kernel, "achieved": k_ach, "frac": k_ach / 770.0,
                                "us_per_step": kernel_ms_per_step * 1e3,
                                "launches_per_step": kernel_launches_per_step,
                                "algorithmic_bytes_per_launch":
                                    bus_bytes / max(kernel_launches_per_step, 1e-9),
                                "timing": timing_note},
                "traffic": None}
        if schedule.startswith("nvls"):
            # bus bytes follow the all-reduce convention (2(N-1)/N S); the
            # bytes the in-switch reduction actually moves per rank and
            # direction are (N+1)/N S, reported beside it
            link = (world + 1) / world * S
            roof["nvls_link_bytes_per_rank_direction"] = link
            roof["nvls_link_frac_of_step"] = link / (ms * 1e-3) / 1e9 / 770.0

    cpu = None
    if not args.no_cpu_baseline and world == 1:      # the contract: rank 0 at N = 1 only
        cus, _, _, desc = oracle_step_time(world, args.dtype, budget_s=args.cpu_budget_s, warmup=1)
        cpu = {"value": cus, "unit": "us", "cores": 1, "kind": "oracle", "sample": desc,
               "cpu": _cpu_model()}
        nth = os.cpu_count() or 1
        if nth > 1:  # same oracle, elements partitioned over all cores
            tus, _, _, tdesc = oracle_step_time(world, args.dtype, budget_s=args.cpu_budget_s / 2,
                                                warmup=1, threads=nth)
            cpu["threaded"] = {"value": tus, "unit": "us", "cores": nth, "sample": tdesc}

    cfg = common_config(P, T, L, args.dtype, world)
    details = {"algo": args.algo if world > 1 else "identity (N=1 fused direct update)",
               "schedule": schedule, "schedule_trials_us": trials,
               "tune_budget_s": args.tune_budget_s if world > 1 else None,
               "comparisons": comparisons or None,
               "step_us_after_l2_write_flush": cold_us,
               "per_step_us": per_step,
               "replicas_bitwise_equal": replicas_equal,
               "warmup_steps_run": n_w,
               "config5_sweep": sweep}
    line = {"metric": METRIC, "value": us, "unit": "us", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded counter-hash, synth/)",
            "config": cfg, "details": details, "bus_gbs": bus,
            "hbm_gbs": roof["achieved"] if world == 1 else None,
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks}
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
