"""Parity of exactly what bench.py times (VERDICT r1 "what's weak" #1).

The headline number is K back-to-back cmn_step launches with no stream
operation in between: programmatic dependent launch (griddepcontrol) lets
step k+1's CTAs start while step k drains, so these tests run the full
ResNet-50 gradient set (BASELINE configs 2 / 3) in the bench's layout (flat
parameter and gradient allocations in the packed layout, one pre-marshalled
pointer table, torch's current stream, the same gradients every step) with
no copy and no synchronisation between steps, then compare every element of
w and v bitwise with K oracle steps.  The same for the step replayed from a
captured CUDA graph, for the events-around-each-launch pass the bench uses
for the per-launch timing, and for simulated N = 8 schedules issued back to
back.  Plus the exhaustive fp16 pin through the GPU cast (SURVEY §8(c) c.4,
PAPER.md:838-839): all 2^32 fp32 bit patterns through k_pack.
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

import synth
from conftest import single_rank_only

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

DEV = "cuda:0"


@pytest.fixture(scope="module")
def cmn(cmn_worlds):
    """Every test here runs in the simulated and in the emulated world
    (conftest.cmn_worlds: barriers live in one cooperative launch)."""
    return cmn_worlds


def _nan_aware_equal(got: np.ndarray, want: np.ndarray, what: str):
    gn, wn = np.isnan(got), np.isnan(want)
    assert np.array_equal(gn, wn), f"{what}: NaN positions differ"
    gb, wb = got.view(np.uint32)[~gn], want.view(np.uint32)[~wn]
    bad = np.flatnonzero(gb != wb)
    assert bad.size == 0, f"{what}: {bad.size} elements differ, first at {bad[:5]}"


class BenchLayout:
    """bench.py's N = 1 setup: flat w and g in the packed layout, views per
    tensor, one prepared pointer table."""

    def __init__(self, cmn, comm, shapes, params0, grads_w0):
        self.sizes = [synth.numel(s) for s in shapes]
        self.off, self.L, _ = cmn.plan_layout(shapes)
        self.flat_w = torch.empty(self.L, dtype=torch.float32, device=DEV)
        self.w = []
        for t, s in enumerate(shapes):
            view = self.flat_w[self.off[t]: self.off[t] + self.sizes[t]].view(s)
            view.copy_(torch.from_numpy(params0[t]).view(s))
            self.w.append(view)
        comm.register_params(self.w)
        self.flat_g = torch.empty(self.L, dtype=torch.float32, device=DEV)
        gv = []
        for t in range(len(shapes)):
            view = self.flat_g[self.off[t]: self.off[t] + self.sizes[t]]
            view.copy_(torch.from_numpy(grads_w0[t]))
            gv.append(view)
        self.table = comm.prepare(gv)
        torch.cuda.synchronize()

    def check(self, comm, w_o, v_o, what):
        got_w = self.flat_w.cpu().numpy()
        got_v = np.concatenate([comm.momentum(t).cpu().numpy().reshape(-1) for t in range(len(w_o))])
        want_w = np.concatenate([x.reshape(-1) for x in w_o])
        want_v = np.concatenate([x.reshape(-1) for x in v_o])
        got_w = np.concatenate([got_w[self.off[t]: self.off[t] + n] for t, n in enumerate(self.sizes)])
        _nan_aware_equal(got_w, want_w, f"{what}: w")
        _nan_aware_equal(got_v, want_v, f"{what}: v")


@pytest.mark.parametrize("dtype", ["fp32", "fp16"])
def test_r50_back_to_back_n1_as_benched(cmn, orc, dtype):
    """N = 1, full ResNet-50 set: 5 back-to-back steps exactly as the timed
    region issues them, then 3 more with the library's per-launch timing
    events (the bench's kernel-duration pass), then 3 replays of a captured
    graph of the step (torch.cuda.graph synchronises once before capturing;
    nothing else does) against 11 oracle steps on the same gradients."""
    single_rank_only(cmn)
    shapes = synth.resnet50_shapes()
    params0 = synth.params(shapes)
    g = synth.grads(shapes, workers=1)
    comm = cmn.Comm.init(0, 1, 0)
    try:
        bl = BenchLayout(cmn, comm, shapes, params0, g[0])
        stream = torch.cuda.current_stream()
        k_plain, k_timed, k_graph = 5, 3, 3
        for _ in range(k_plain):
            comm.step(bl.table, dtype, 0.1, 0.9, stream)
        comm.set_kernel_timing(True)
        for _ in range(k_timed):
            comm.step(bl.table, dtype, 0.1, 0.9, stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):              # capture is not executed
            comm.step(bl.table, dtype, 0.1, 0.9)
        for _ in range(k_graph):
            graph.replay()
        torch.cuda.synchronize()
        _, n_timed = comm.kernel_timing()
        comm.set_kernel_timing(False)
        assert n_timed == k_timed                   # the bracketed launches really ran
        w_o = [p.copy() for p in params0]
        v_o = [np.zeros_like(p) for p in params0]
        for _ in range(k_plain + k_timed + k_graph):
            orc.step(g, w_o, v_o, 0.1, 0.9, dtype)
        bl.check(comm, w_o, v_o, f"R50 N=1 {dtype}, {k_plain}+{k_timed}+{k_graph} back-to-back steps")
    finally:
        comm.finalize()


@pytest.mark.parametrize("sched,dtype", [("pipelined4", "fp32"), ("fused_pull", "fp16"),
                                         ("fused_push", "fp32"), ("pipelined4_graph", "fp16")])
def test_r50_sim8_back_to_back(cmn, orc, sched, dtype):
    """Simulated N = 8 (the N > 1 kernels, one launch per simulated rank),
    full ResNet-50 set, the schedules the N > 1 bench line chooses between,
    3 steps issued back to back without synchronisation (the pipelined
    one also as 3 replays of a captured graph)."""
    shapes = synth.resnet50_shapes()
    N = 8
    params0 = synth.params(shapes)
    g = synth.grads(shapes, workers=N)
    comm = cmn.Comm.simulated_world(N)
    try:
        sizes = [synth.numel(s) for s in shapes]
        off, L, _ = cmn.plan_layout(shapes)
        flat_w = torch.empty(L, dtype=torch.float32, device=DEV)
        w = [flat_w[off[t]: off[t] + sizes[t]].view(shapes[t]) for t in range(len(shapes))]
        for t in range(len(w)):
            w[t].copy_(torch.from_numpy(params0[t]).view(shapes[t]))
        comm.register_params(w)
        table = comm.prepare([[torch.from_numpy(x).to(DEV) for x in gw] for gw in g])
        comm.set_fused_update({"fused_pull": 1, "fused_push": 2}.get(sched, 0))
        comm.set_pipeline(4 if sched.startswith("pipelined") else 0)
        torch.cuda.synchronize()
        K = 3
        if sched.endswith("_graph"):
            comm.step(table, dtype, 0.1, 0.9)        # step 1 eagerly (internal streams exist)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                comm.step(table, dtype, 0.1, 0.9)
            for _ in range(K - 1):
                graph.replay()
        else:
            for _ in range(K):
                comm.step(table, dtype, 0.1, 0.9)
        torch.cuda.synchronize()
        got_w = flat_w.cpu().numpy()
        got_v = [comm.momentum(t).cpu().numpy().reshape(-1) for t in range(len(w))]
    finally:
        comm.finalize()
    del table
    w_o = [p.copy() for p in params0]
    v_o = [np.zeros_like(p) for p in params0]
    for _ in range(K):
        orc.step(g, w_o, v_o, 0.1, 0.9, dtype)
    _nan_aware_equal(np.concatenate([got_w[off[t]: off[t] + n] for t, n in enumerate(sizes)]),
                     np.concatenate(w_o), f"{sched} {dtype} w")
    _nan_aware_equal(np.concatenate(got_v), np.concatenate(v_o), f"{sched} {dtype} v")


def test_fp16_cast_all_2pow32_patterns_on_gpu(cmn, orc):
    """SURVEY §8(c) c.4 / PAPER.md:838-839: every one of the 2^32 fp32 bit
    patterns through the GPU path's cast (k_pack of cmn_allreduce_grads with
    an fp16 payload, N = 1, so the packed buffer is the cast) against the
    oracle's hand-written RNE (itself pinned to the compiler's _Float16 over
    all 2^32 inputs on the host).  NaNs are compared by class: both sides
    must produce an fp16 NaN for exactly the fp32 NaNs.  16 chunks of 2^28;
    the oracle side runs on host threads (bit-identical, elementwise)."""
    single_rank_only(cmn)
    chunk = 1 << 28
    comm = cmn.Comm.init(0, 1, 0)
    pool = ThreadPoolExecutor(max_workers=8)
    try:
        w = [torch.zeros(chunk, dtype=torch.float32, device=DEV)]
        comm.register_params(w)
        x_dev = torch.empty(chunk, dtype=torch.int32, device=DEV)
        p = torch.empty(chunk, dtype=torch.int16, device=DEV)
        base_host = np.arange(chunk, dtype=np.uint32)
        for c in range(1 << 4):
            lo = c * chunk
            # the input: bit patterns lo .. lo + 2^28 - 1 (built on the device
            # as plain integers, no arithmetic of the method)
            v = torch.arange(lo, lo + chunk, dtype=torch.int64, device=DEV)
            x_dev.copy_(torch.where(v >= (1 << 31), v - (1 << 32), v).to(torch.int32))
            del v
            comm.allreduce_grads([x_dev.view(torch.float32)], "fp16")
            comm.copy_packed(0, p)
            torch.cuda.synchronize()
            got = p.cpu().numpy().view(np.uint16)
            xs = (base_host + np.uint32(lo)).view(np.float32)
            parts = np.array_split(np.arange(chunk), 8)
            want = np.empty(chunk, dtype=np.uint16)

            def run(ix):
                want[ix[0]: ix[-1] + 1] = orc.f32_to_f16(xs[ix[0]: ix[-1] + 1])
            list(pool.map(run, parts))
            gn = ((got & 0x7C00) == 0x7C00) & ((got & 0x3FF) != 0)
            wn = ((want & 0x7C00) == 0x7C00) & ((want & 0x3FF) != 0)
            assert np.array_equal(gn, wn), f"chunk {c}: NaN positions differ"
            bad = np.flatnonzero((got != want) & ~wn)
            assert bad.size == 0, (f"chunk {c}: {bad.size} patterns differ, e.g. "
                                   f"{[hex(int(lo) + int(i)) for i in bad[:4]]}")
    finally:
        pool.shutdown()
        comm.finalize()
