"""The cross-rank barrier protocol on ONE GPU without separate launches that
wait on one another: cmn_init_emulated plays all N ranks in one process and
runs each one-shot / two-shot all-reduce as ONE cooperative launch of N x G
blocks (block r * G + b is CTA b of rank r, every block co-resident), with
the barriers live -- flag pads, per-rank per-CTA epochs, call tags, the
two-shot mid barrier, the one-shot end barrier, timeouts and poison flags.
(B200_PROFILING.md: ranks that spin on each other's flags must not be
separate launches on one GPU; emulate them as one kernel over all ranks'
data, cooperative if its blocks wait on one another.)

Everything is compared bitwise with the CPU oracle (§6.1.2:
sum over workers, divide by the number of replicas, update each replica;
readings R2/R3/R6 in DESIGN.md §3): every rank's reduced buffer and the
parameters / momentum after every step."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

DEV = "cuda:0"
# ragged shapes spanning several 4096-element work items and tails, plus the MLP
RAGGED = [(1,), (3,), (4097,), (8191,), (12289,), (65,), (100, 784), (100,), (10, 100), (10,)]


@pytest.fixture(scope="module")
def cmn():
    from paper_1908_00213_b200 import build
    build.build()
    from paper_1908_00213_b200 import cmn as m
    return m


def _u32(x):
    return np.ascontiguousarray(x).view(np.uint32)


def _same(got, want, what):
    gn, wn = np.isnan(got), np.isnan(want)
    assert np.array_equal(gn, wn), f"{what}: NaN positions differ"
    bad = _u32(got)[~gn] != _u32(want)[~wn]
    assert not bad.any(), f"{what}: {int(bad.sum())} elements differ"


def _emulated(cmn, N, algo, pieces=0):
    comm = cmn.Comm.emulated_world(N)
    comm.set_algo(algo)
    comm.set_pipeline(pieces)
    return comm


def _oracle_steps(orc, shapes, N, dtype, steps, lr, mu, value_set="random"):
    """Per step: the oracle's reduced buffer (as float32) and w, v after it."""
    sizes = [synth.numel(s) for s in shapes]
    off, L = orc.layout(sizes)
    w = synth.params(shapes, value_set=value_set)
    v = [np.zeros_like(x) for x in w]
    out = []
    for k in range(steps):
        g = synth.grads(shapes, workers=N, step=k, value_set=value_set)
        packed = [orc.pack(gw, off, L, dtype) for gw in g]
        red = orc.reduce_tree(packed, dtype)
        orc.update_momentum_sgd(red, dtype, N, lr, mu, off, w, v)
        red32 = red if dtype == "fp32" else orc.f16_to_f32(red)
        out.append({"reduced": np.asarray(red32, dtype=np.float32), "w": [x.copy() for x in w],
                    "v": [x.copy() for x in v]})
    return out, L


def _dev_grads(shapes, N, step, value_set="random"):
    return [[torch.from_numpy(g).to(DEV) for g in gw]
            for gw in synth.grads(shapes, workers=N, step=step, value_set=value_set)]


@pytest.mark.parametrize("N", [2, 3, 5, 8])
@pytest.mark.parametrize("dtype", ["fp32", "fp16"])
@pytest.mark.parametrize("algo", ["oneshot", "twoshot"])
def test_emulated_world_bitexact(cmn, orc, N, dtype, algo):
    """Barriers live, every rank's reduced buffer and w, v after 3 steps
    (so the per-CTA epochs advance) bit-exact vs the oracle; ONE launch per
    all-reduce (all ranks in one cooperative grid)."""
    shapes, lr, mu = RAGGED, 0.1, 0.9
    want, L = _oracle_steps(orc, shapes, N, dtype, 3, lr, mu)
    comm = _emulated(cmn, N, algo)
    try:
        w = [torch.from_numpy(p).to(DEV) for p in synth.params(shapes)]
        comm.register_params(w)
        tdt = torch.float32 if dtype == "fp32" else torch.float16
        for k in range(3):
            n0 = comm.kernel_launches
            comm.allreduce_grads(_dev_grads(shapes, N, k), dtype)
            # N packs (one per simulated rank's gradients) + ONE all-reduce launch
            assert comm.kernel_launches - n0 == N + 1
            for r in range(N):
                q = torch.empty(L, dtype=tdt, device=DEV)
                comm.copy_reduced(r, q)
                _same(q.float().cpu().numpy(), want[k]["reduced"], f"step {k} reduced rank {r}")
            comm.update_momentum_sgd(lr, mu)
            torch.cuda.synchronize()
            for t in range(len(w)):
                _same(w[t].cpu().numpy().reshape(-1), want[k]["w"][t], f"step {k} w[{t}]")
                _same(comm.momentum(t).cpu().numpy().reshape(-1), want[k]["v"][t], f"step {k} v[{t}]")
        comm.poll_error()
    finally:
        comm.finalize()


@pytest.mark.slow
@pytest.mark.parametrize("dtype", ["fp32", "fp16"])
@pytest.mark.parametrize("sched", ["serial", "pipelined4", "fused", "sharded"])
def test_emulated_r50_n8_back_to_back(cmn, orc, dtype, sched):
    """The full ResNet-50 gradient set, 8 emulated ranks, barriers live, 3
    steps issued back to back: serial two-shot (start + mid barrier), the
    pipelined 4-piece schedule (all-reduces on the internal stream), the
    fused pull schedule (reduce-scatter, then the fused all-gather + update
    with its start barrier) and the sharded step (reduce-scatter, own-chunk
    update, parameter all-gather).  w bit-exact vs 3 oracle steps, and v too
    (the sharded step keeps v on the chunk owner: one replica holds all)."""
    shapes, N, lr, mu, K = synth.resnet50_shapes(), 8, 0.1, 0.9, 3
    w0 = synth.params(shapes)
    wo, vo = [x.copy() for x in w0], [np.zeros_like(x) for x in w0]
    for k in range(K):
        orc.step(synth.grads(shapes, workers=N, step=k), wo, vo, lr, mu, dtype)
    comm = _emulated(cmn, N, "twoshot", 4 if sched == "pipelined4" else 0)
    try:
        comm.set_fused_update(1 if sched == "fused" else 0)
        w = [torch.from_numpy(p).to(DEV) for p in w0]
        comm.register_params(w)
        tables = [comm.prepare([g for gw in _dev_grads(shapes, N, k) for g in gw]) for k in range(K)]
        torch.cuda.synchronize()
        n0 = comm.kernel_launches
        for k in range(K):
            (comm.step_sharded if sched == "sharded" else comm.step)(tables[k], dtype, lr, mu)
        torch.cuda.synchronize()
        comm.poll_error()
        if sched == "fused":      # per step: N packs + ONE reduce-scatter + ONE all-gather/update
            assert comm.kernel_launches - n0 == K * (N + 2)
        for t in range(len(w)):
            _same(w[t].cpu().numpy().reshape(-1), wo[t], f"w[{t}]")
            _same(comm.momentum(t).cpu().numpy().reshape(-1), vo[t], f"v[{t}]")
    finally:
        comm.finalize()


def test_emulated_many_calls_epochs(cmn, orc):
    """60 steps alternating algorithm, payload dtype and pipeline pieces (so
    the barrier tags change from call to call and the per-CTA epochs run
    far), each bit-exact vs the oracle replaying the same sequence."""
    shapes, N, lr, mu = synth.mlp_shapes(), 4, 0.05, 0.9
    sizes = [synth.numel(s) for s in shapes]
    off, L = orc.layout(sizes)
    w0 = synth.params(shapes)
    wo, vo = [x.copy() for x in w0], [np.zeros_like(x) for x in w0]
    comm = cmn.Comm.emulated_world(N)
    try:
        w = [torch.from_numpy(p).to(DEV) for p in w0]
        comm.register_params(w)
        rng = np.random.default_rng(190800213)
        for k in range(60):
            algo = ["oneshot", "twoshot"][rng.integers(2)]
            dtype = ["fp32", "fp16"][rng.integers(2)]
            pieces = [0, 2, 3][rng.integers(3)]
            comm.set_algo(algo)
            comm.set_pipeline(pieces)
            comm.step(_dev_grads(shapes, N, k % 7), dtype, lr, mu)
            orc.step(synth.grads(shapes, workers=N, step=k % 7), wo, vo, lr, mu, dtype)
        torch.cuda.synchronize()
        comm.poll_error()
        for t in range(len(w)):
            _same(w[t].cpu().numpy().reshape(-1), wo[t], f"w[{t}]")
            _same(comm.momentum(t).cpu().numpy().reshape(-1), vo[t], f"v[{t}]")
    finally:
        comm.finalize()


def test_emulated_graph_replay(cmn, orc):
    """The pipelined step captured into a CUDA graph (cooperative all-reduce
    launches inside it) and replayed: barrier epochs live on the device, so
    replays pair correctly; 1 eager + 3 replays == 4 oracle steps."""
    shapes, N, lr, mu = RAGGED, 4, 0.1, 0.9
    w0 = synth.params(shapes)
    wo, vo = [x.copy() for x in w0], [np.zeros_like(x) for x in w0]
    g = synth.grads(shapes, workers=N, step=0)
    for _ in range(4):
        orc.step(g, wo, vo, lr, mu, "fp32")
    comm = _emulated(cmn, N, "twoshot", 2)
    try:
        w = [torch.from_numpy(p).to(DEV) for p in w0]
        comm.register_params(w)
        table = comm.prepare([x for gw in _dev_grads(shapes, N, 0) for x in gw])
        comm.step(table, "fp32", lr, mu, torch.cuda.current_stream())
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            comm.step(table, "fp32", lr, mu)
        for _ in range(3):
            graph.replay()
        torch.cuda.synchronize()
        comm.poll_error()
        for t in range(len(w)):
            _same(w[t].cpu().numpy().reshape(-1), wo[t], f"w[{t}]")
            _same(comm.momentum(t).cpu().numpy().reshape(-1), vo[t], f"v[{t}]")
    finally:
        comm.finalize()


@pytest.mark.parametrize("fault,code", [("CMN_TEST_EMUL_ABSENT_RANK", 6), ("CMN_TEST_EMUL_MISMATCH_RANK", 5)])
@pytest.mark.parametrize("algo", ["oneshot", "twoshot", "pipelined3", "fused", "sharded"])
def test_emulated_fault_leaves_state_untouched(cmn, monkeypatch, fault, code, algo):
    """A rank that never arrives (its peers' barriers time out: CMN_ERR_TIMEOUT)
    or posts another call tag (CMN_ERR_MISMATCH) in the step's first
    all-reduce kernel: the failed step leaves w and v bit-identical (every
    CTA skips its stores; the later kernels of the step -- the update, the
    fused all-gather + update, the sharded chunk update and parameter
    all-gather -- see the device error word or post poison and touch
    nothing), the error surfaces on the next call, and the communicator
    stays failed."""
    from paper_1908_00213_b200.cmn import CmnError
    monkeypatch.setenv(fault, "2")
    shapes, N = RAGGED, 4
    comm = _emulated(cmn, N, "oneshot" if algo == "oneshot" else "twoshot",
                     3 if algo == "pipelined3" else 0)
    try:
        comm.set_timeout(300)
        comm.set_fused_update(1 if algo == "fused" else 0)
        w = [torch.from_numpy(p).to(DEV) for p in synth.params(shapes)]
        comm.register_params(w)
        w_before = [x.clone() for x in w]
        (comm.step_sharded if algo == "sharded" else comm.step)(_dev_grads(shapes, N, 0), "fp32", 0.1, 0.9)
        torch.cuda.synchronize()
        for t in range(len(w)):
            assert torch.equal(w[t].view(torch.int32), w_before[t].view(torch.int32)), f"w[{t}] changed"
            assert not comm.momentum(t).any(), f"v[{t}] changed"
        with pytest.raises(CmnError) as ei:
            comm.step(_dev_grads(shapes, N, 1), "fp32", 0.1, 0.9)
        assert ei.value.status == code, ei.value
        with pytest.raises(CmnError):
            comm.poll_error()
    finally:
        comm.finalize()


def test_emulated_reregistration_structure_changes(cmn, orc):
    """Define-by-Run at N > 1 ("model structure can be
    changed at any iteration dynamically"): the registered structure changes
    between iterations (MLP depth 3 -> 3 -> 4 -> 4 -> 3, each model keeping
    its own parameters), every change a re-registration that re-plans the
    layout and resets momentum (reading R7); 4 emulated ranks with the
    barriers live across re-registrations.  Each model's parameters and the
    final momentum bit-exact vs the oracle replaying the same sequence."""
    def shapes_of(depth):
        dims = [784] + [100] * (depth - 1) + [10]
        out = []
        for i in range(depth):
            out += [(dims[i + 1], dims[i]), (dims[i + 1],)]
        return out

    N, lr, mu, depths = 4, 0.05, 0.9, [3, 3, 4, 4, 3]
    models = {d: synth.params(shapes_of(d), seed=40 + d) for d in sorted(set(depths))}
    dev_w = {d: [torch.from_numpy(p.copy()).to(DEV) for p in models[d]] for d in models}
    w_o = {d: [p.copy() for p in models[d]] for d in models}
    comm = cmn.Comm.emulated_world(N)
    try:
        comm.set_algo("twoshot")
        cur, v_o = None, None
        for it, d in enumerate(depths):
            shapes = shapes_of(d)
            if d != cur:
                comm.register_params(dev_w[d])
                v_o = [np.zeros_like(x) for x in w_o[d]]
                cur = d
            comm.step(_dev_grads(shapes, N, it), "fp32", lr, mu)
            orc.step(synth.grads(shapes, workers=N, step=it), w_o[d], v_o, lr, mu, "fp32")
        torch.cuda.synchronize()
        comm.poll_error()
        for d in models:
            for t in range(len(models[d])):
                _same(dev_w[d][t].cpu().numpy().reshape(-1), w_o[d][t], f"depth {d} w[{t}]")
        for t in range(len(v_o)):
            _same(comm.momentum(t).cpu().numpy().reshape(-1), v_o[t], f"v[{t}]")
    finally:
        comm.finalize()


def _run_twoshot_steps(cmn, shapes, N, steps):
    """Every rank's reduced buffer (float32 values) after each of `steps`
    two-shot all-reduces in the emulated world; w, v after the last step."""
    comm = _emulated(cmn, N, "twoshot")
    try:
        w = [torch.from_numpy(p).to(DEV) for p in synth.params(shapes)]
        comm.register_params(w)
        L = comm.layout()[1]
        red = []
        for k in range(steps):
            comm.allreduce_grads(_dev_grads(shapes, N, k), "fp32")
            per = []
            for r in range(N):
                q = torch.empty(L, dtype=torch.float32, device=DEV)
                comm.copy_reduced(r, q)
                per.append(q)
            comm.update_momentum_sgd(0.1, 0.9)
            torch.cuda.synchronize()
            red.append([q.cpu().numpy() for q in per])
        comm.poll_error()
        return red
    finally:
        comm.finalize()


def test_emulated_slow_rank_mid_barrier(cmn, orc, monkeypatch):
    """Rank 3's blocks stall 2 ms after the start barrier, before reducing
    their chunk: every other rank finishes its reduce-scatter and must wait
    at the two-shot mid barrier for rank 3's chunk before gathering it.
    Every rank's reduced buffer stays bit-exact over 3 steps."""
    monkeypatch.setenv("CMN_TEST_EMUL_SLOW_RANK", "3")
    monkeypatch.setenv("CMN_TEST_ONESHOT_DELAY_US", "2000")
    shapes, N = RAGGED, 4
    want, _ = _oracle_steps(orc, shapes, N, "fp32", 3, 0.1, 0.9)
    got = _run_twoshot_steps(cmn, shapes, N, 3)
    for k in range(3):
        for r in range(N):
            _same(got[k][r], want[k]["reduced"], f"step {k} rank {r}")


def test_emulated_negative_control_without_mid_barrier(cmn, orc, monkeypatch):
    """The same slow rank with the mid barrier compiled out of the call
    (CMN_TEST_EMUL_SKIP_MID): the other ranks gather rank 3's chunk before
    rank 3 has reduced it and end up with a wrong sum -- the emulated world
    does expose a missing cross-rank ordering (the test above is not
    vacuous)."""
    monkeypatch.setenv("CMN_TEST_EMUL_SLOW_RANK", "3")
    monkeypatch.setenv("CMN_TEST_ONESHOT_DELAY_US", "2000")
    monkeypatch.setenv("CMN_TEST_EMUL_SKIP_MID", "1")
    shapes, N = RAGGED, 4
    want, _ = _oracle_steps(orc, shapes, N, "fp32", 3, 0.1, 0.9)
    got = _run_twoshot_steps(cmn, shapes, N, 3)
    bad = sum(int(np.count_nonzero(_u32(got[k][r]) != _u32(want[k]["reduced"])))
              for k in range(3) for r in range(N))
    assert bad > 0, "without the mid barrier the gathered chunks should be stale"


def test_emulated_random_schedule_stress(cmn, orc):
    """80 steps, 4 emulated ranks, barriers live, the schedule redrawn every
    step from serial one-/two-shot, pipelined (2 / 3 pieces), fused pull,
    fused push, sharded and bucketed, with the payload dtype and the
    collective / update grids redrawn too (barrier kernels of different
    kinds, tags and CTA counts interleave, so per-CTA epochs of different
    indices advance at different rates): w and v bit-exact vs the oracle
    replaying the same 80 steps."""
    shapes, N, lr, mu = synth.mlp_shapes() + RAGGED, 4, 0.05, 0.9
    w0 = synth.params(shapes)
    wo, vo = [x.copy() for x in w0], [np.zeros_like(x) for x in w0]
    comm = cmn.Comm.emulated_world(N)
    try:
        w = [torch.from_numpy(p).to(DEV) for p in w0]
        comm.register_params(w)
        nb = comm.plan_buckets(1 << 16)
        rng = np.random.default_rng(20261018)
        scheds = ["oneshot", "twoshot", "pipelined2", "pipelined3", "fused", "push", "sharded", "buckets"]
        for k in range(80):
            sched = scheds[rng.integers(len(scheds))]
            dtype = ["fp32", "fp16"][rng.integers(2)]
            ctas = [0, 16, 64][rng.integers(3)]
            comm.set_ctas(ctas, [0, 148][rng.integers(2)])
            comm.set_algo("oneshot" if sched == "oneshot" else "twoshot")
            comm.set_pipeline({"pipelined2": 2, "pipelined3": 3}.get(sched, 0))
            comm.set_fused_update({"fused": 1, "push": 2}.get(sched, 0))
            gd = _dev_grads(shapes, N, k % 5)
            if sched == "sharded":
                comm.step_sharded(gd, dtype, lr, mu)
            elif sched == "buckets":
                for b in range(nb):
                    comm.allreduce_bucket(b, gd, dtype)
                for b in range(nb):
                    comm.update_bucket(b, lr, mu)
            else:
                comm.step(gd, dtype, lr, mu)
            orc.step(synth.grads(shapes, workers=N, step=k % 5), wo, vo, lr, mu, dtype)
        torch.cuda.synchronize()
        comm.poll_error()
        for t in range(len(w)):
            _same(w[t].cpu().numpy().reshape(-1), wo[t], f"w[{t}]")
            _same(comm.momentum(t).cpu().numpy().reshape(-1), vo[t], f"v[{t}]")
    finally:
        comm.finalize()


@pytest.mark.parametrize("N", [2, 4, 8])
@pytest.mark.parametrize("dtype", ["fp32", "fp16"])
def test_emulated_push_form(cmn, orc, N, dtype):
    """The fused push step in the emulated world (every rank's gradient
    pointers fit one launch: N * T <= 256): ONE cooperative pack + push
    launch (each rank's blocks cast its gradients into every owner's inbox
    slot), ONE cooperative inbox reduce-scatter, ONE cooperative all-gather
    + update -- 3 launches per step, barriers live -- and w, v bit-exact vs
    3 oracle steps."""
    shapes, lr, mu = synth.mlp_shapes() + RAGGED, 0.1, 0.9
    w0 = synth.params(shapes)
    wo, vo = [x.copy() for x in w0], [np.zeros_like(x) for x in w0]
    for k in range(3):
        orc.step(synth.grads(shapes, workers=N, step=k), wo, vo, lr, mu, dtype)
    comm = _emulated(cmn, N, "twoshot")
    try:
        comm.set_fused_update(2)
        w = [torch.from_numpy(p).to(DEV) for p in w0]
        comm.register_params(w)
        for k in range(3):
            n0 = comm.kernel_launches
            comm.step(_dev_grads(shapes, N, k), dtype, lr, mu)
            assert comm.kernel_launches - n0 == 3
        torch.cuda.synchronize()
        comm.poll_error()
        for t in range(len(w)):
            _same(w[t].cpu().numpy().reshape(-1), wo[t], f"w[{t}]")
            _same(comm.momentum(t).cpu().numpy().reshape(-1), vo[t], f"v[{t}]")
    finally:
        comm.finalize()
