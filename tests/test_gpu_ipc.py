"""The real multi-process path (cmn_init: CUDA-IPC peer mapping, per-CTA
release/acquire barriers across processes), one process per GPU: rank r on
device r.  Each process owns its buffers, peers read them through IPC
mappings over NVSwitch.  Results are compared bit-exact with the oracle and
across ranks (replica consistency); every spin is bounded by the
device timeout.

These tests need one GPU per rank (conftest.require_gpus_for_ranks): ranks
whose kernels spin on each other's flags must never be separate launches on
one GPU (B200_PROFILING.md).  On a one-GPU box they skip; the barrier
protocol is then covered by tests/test_gpu_emulated.py (all ranks in one
cooperative launch, barriers live)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import synth

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, dtype, algo, steps, q, mode, pieces=0):
    import torch
    import torch.distributed as dist

    from paper_1908_00213_b200 import cmn
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if mode.startswith("slow_peer") and rank == 1:
        # fault injection: this rank's one-shot CTAs stall 20 ms after their
        # start barrier, so rank 0 races ahead into its next step
        os.environ["CMN_TEST_ONESHOT_DELAY_US"] = "20000"
    try:
        dev = rank % torch.cuda.device_count()          # one GPU per rank
        torch.cuda.set_device(dev)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        shapes = synth.mlp_shapes()
        digest = mode.startswith("r50:")          # full ResNet-50 set: return hashes
        if digest:
            shapes, mode = synth.resnet50_shapes(), mode[4:]
        if mode == "mismatch" and rank == 1:
            shapes = shapes[:-1] + [(11,)]
        comm = cmn.Comm.init(rank, world, dev, dist.group.WORLD)
        comm.set_timeout(3000 if mode == "skip" else 60000)
        w = [torch.from_numpy(p).cuda() for p in synth.params(shapes)]
        try:
            comm.register_params(w)
        except cmn.CmnError as e:
            q.put((rank, "error", e.status_name))
            return
        if mode == "setup_alt":
            # NVLS / NCCL resources are created collectively: whatever the box
            # supports, every rank must get the same outcome (never a hang)
            try:
                comm.set_algo(algo)
                q.put((rank, "ok"))
            except cmn.CmnError as e:
                q.put((rank, "error", e.status_name))
            dist.barrier()
            comm.finalize()
            return
        comm.set_algo(algo)
        comm.set_pipeline(pieces + (rank if mode == "piece_mismatch" else 0))
        comm.set_fused_update(2 if mode in ("push", "graph_push") else mode in ("fused", "graph_fused"))
        if mode == "capture_unpipelined":
            g0 = [torch.from_numpy(x).cuda() for x in synth.grads(shapes, workers=world)[rank]]
            comm.allreduce_grads(g0, dtype)          # eager warm-up is fine
            comm.update_momentum_sgd(0.1, 0.9)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            try:
                with torch.cuda.graph(graph):
                    comm.allreduce_grads(g0, dtype)
                q.put((rank, "ok-unexpected"))
            except cmn.CmnError as e:
                q.put((rank, "error", e.status_name))
            dist.barrier()
            return
        if mode in ("graph", "graph_sharded", "graph_fused", "graph_push", "slow_peer_graph"):
            # step 0 eagerly (creates internal streams), then capture ONE step
            # into a CUDA graph and replay it for steps 1.. with fresh grads
            # copied into the captured buffers.
            gs = [torch.from_numpy(x).cuda() for x in synth.grads(shapes, workers=world, step=0)[rank]]
            fn = comm.step_sharded if mode == "graph_sharded" else comm.step
            fn(gs, dtype, 0.1, 0.9)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                fn(gs, dtype, 0.1, 0.9)
            for s in range(1, steps):
                for dst, x in zip(gs, synth.grads(shapes, workers=world, step=s)[rank]):
                    dst.copy_(torch.from_numpy(x))
                graph.replay()
            steps = 0
        snap = None
        for s in range(steps):
            g = [torch.from_numpy(x).cuda() for x in synth.grads(shapes, workers=world, step=s)[rank]]
            if mode in ("skip", "piece_mismatch"):
                torch.cuda.synchronize()
                snap = [np.concatenate([x.cpu().numpy().reshape(-1) for x in w]),
                        np.concatenate([comm.momentum(t).cpu().numpy().reshape(-1) for t in range(len(w))])]
            if mode == "skip" and rank == 1 and s == 1:
                continue                              # fault injection: rank 1 skips a collective
            if mode == "reregister" and s == 1:
                comm.register_params(w)               # collective; resets momentum (reading R7)
            if mode == "stress":
                # long run, schedule / grid / algorithm drawn per step from a
                # seed shared by all ranks
                import random
                rnd = random.Random(1000 + s)
                sched = rnd.choice(["serial1", "serial2", "pipelined", "pull", "push", "graphless"])
                comm.set_algo("oneshot" if sched == "serial1" else "twoshot")
                comm.set_fused_update({"pull": 1, "push": 2}.get(sched, 0))
                comm.set_pipeline(rnd.choice([2, 3, 5]) if sched == "pipelined" else 0)
                comm.set_ctas(rnd.choice([0, 1, 7, 148]), rnd.choice([0, 3, 64]))
                if sched == "graphless":
                    comm.allreduce_grads(g, dtype)
                    comm.update_momentum_sgd(0.1, 0.9)
                else:
                    comm.step(g, dtype, 0.1, 0.9)
            elif mode == "adam":
                comm.step_adam(g, dtype, 1e-3, 0.9, 0.999, 1e-8, s + 1)   # pipelined when pieces >= 2
            elif mode == "host":
                # e2e form through pinned host buffers (pipelined: H2D/D2H per piece)
                sizes = [x.numel() for x in w]
                off, L = cmn.plan_layout(shapes)[:2]
                hg = torch.zeros(L, dtype=torch.float32).pin_memory()
                for t, x in enumerate(g):
                    hg[off[t]: off[t] + sizes[t]].copy_(x.reshape(-1).cpu())
                hw = torch.full((L,), float("nan"), dtype=torch.float32).pin_memory()
                comm.step_host_packed(hg, hw, dtype, 0.1, 0.9)
                torch.cuda.synchronize()
                for t, x in enumerate(w):
                    if not torch.equal(hw[off[t]: off[t] + sizes[t]].view(torch.int32),
                                       x.reshape(-1).cpu().view(torch.int32)):
                        raise RuntimeError(f"host params of tensor {t} differ from device params")
            elif mode == "mixed":
                # the schedule and the grid sizes change every step, identically
                # on every rank: per-CTA barrier epochs must stay paired
                fused, pcs, ctas = [(1, 0, (5, 3)), (0, 2, (9, 0)), (2, 0, (3, 9)),
                                    (0, 0, (0, 0)), (1, 0, (1, 700)), (2, 0, (0, 0))][s % 6]
                comm.set_fused_update(fused)
                comm.set_pipeline(pcs)
                comm.set_ctas(*ctas)
                if fused or pcs:
                    comm.step(g, dtype, 0.1, 0.9)
                else:
                    comm.allreduce_grads(g, dtype)
                    comm.update_momentum_sgd(0.1, 0.9)
            elif mode == "sharded":
                comm.step_sharded(g, dtype, 0.1, 0.9)  # RS -> own-chunk update -> param all-gather
            elif mode in ("fused", "push"):
                comm.step(g, dtype, 0.1, 0.9)         # RS (pulled / pushed) -> fused all-gather + update
            elif pieces:
                comm.step(g, dtype, 0.1, 0.9)         # pipelined schedule, 2 streams
            else:
                comm.allreduce_grads(g, dtype)
                comm.update_momentum_sgd(0.1, 0.9)
        torch.cuda.synchronize()
        try:
            comm.poll_error()
            wb = np.concatenate([x.cpu().numpy().reshape(-1) for x in w])
            vb = np.concatenate([comm.momentum(t).cpu().numpy().reshape(-1) for t in range(len(w))])
            if digest:
                import hashlib
                q.put((rank, "ok", hashlib.sha256(wb.tobytes()).hexdigest(),
                       hashlib.sha256(vb.tobytes()).hexdigest()))
            else:
                q.put((rank, "ok", wb.tobytes(), vb.tobytes()))
        except cmn.CmnError as e:
            if snap is not None:
                # the failed call must leave w and v exactly as they were
                wb = np.concatenate([x.cpu().numpy().reshape(-1) for x in w])
                vb = np.concatenate([comm.momentum(t).cpu().numpy().reshape(-1) for t in range(len(w))])
                same = wb.tobytes() == snap[0].tobytes() and vb.tobytes() == snap[1].tobytes()
                q.put((rank, "error", e.status_name, same))
            else:
                q.put((rank, "error", e.status_name))
        dist.barrier()            # no rank frees its IPC-exported buffers while a peer may read them
        comm.finalize()
    except Exception as e:  # noqa: BLE001
        q.put((rank, "exc", repr(e)))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def _run(world, dtype, algo, steps=2, mode="same", pieces=0):
    from conftest import require_gpus_for_ranks
    require_gpus_for_ranks(world)
    from paper_1908_00213_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, dtype, algo, steps, q, mode, pieces))
          for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in ps:
        p.join(timeout=120)
    return sorted(res, key=lambda r: r[0])


@pytest.mark.parametrize("world,dtype,algo,pieces", [(2, "fp32", "oneshot", 0), (2, "fp16", "twoshot", 0),
                                                     (3, "fp32", "twoshot", 0), (3, "fp16", "oneshot", 0),
                                                     (2, "fp32", "twoshot", 3), (3, "fp16", "twoshot", 2)])
def test_ipc_multiprocess_parity(orc, world, dtype, algo, pieces):
    res = _run(world, dtype, algo, pieces=pieces)
    assert all(r[1] == "ok" for r in res), res
    shapes = synth.mlp_shapes()
    w = synth.params(shapes)
    v = [np.zeros_like(x) for x in w]
    for s in range(2):
        orc.step(synth.grads(shapes, workers=world, step=s), w, v, 0.1, 0.9, dtype)
    want_w = np.concatenate(w).view(np.uint32)
    want_v = np.concatenate(v).view(np.uint32)
    for r in res:
        assert np.array_equal(np.frombuffer(r[2], np.uint32), want_w), f"rank {r[0]} w"
        assert np.array_equal(np.frombuffer(r[3], np.uint32), want_v), f"rank {r[0]} v"


@pytest.mark.parametrize("world,dtype", [(2, "fp32"), (3, "fp16")])
def test_ipc_sharded_update(orc, world, dtype):
    """NEXT-4 across processes: every rank ends with the oracle's w (bitwise);
    the momentum is current on each rank's own chunk."""
    from paper_1908_00213_b200 import cmn
    res = _run(world, dtype, "twoshot", mode="sharded")
    assert all(r[1] == "ok" for r in res), res
    shapes = synth.mlp_shapes()
    w = synth.params(shapes)
    v = [np.zeros_like(x) for x in w]
    for s in range(2):
        orc.step(synth.grads(shapes, workers=world, step=s), w, v, 0.1, 0.9, dtype)
    want_w = np.concatenate(w).view(np.uint32)
    sizes = [x.size for x in w]
    off, L = orc.layout(sizes)
    starts, ends = cmn.plan_chunks(L, world)
    vflat = np.concatenate(v).view(np.uint32)
    for r in res:
        assert np.array_equal(np.frombuffer(r[2], np.uint32), want_w), f"rank {r[0]} w"
        got_v = np.frombuffer(r[3], np.uint32)
        pos = 0
        for t, n in enumerate(sizes):          # elements (t, k) with packed index in own chunk
            j = off[t] + np.arange(n)
            own = (j >= starts[r[0]]) & (j < ends[r[0]])
            assert np.array_equal(got_v[pos:pos + n][own], vflat[pos:pos + n][own]), f"rank {r[0]} v[{t}]"
            pos += n


@pytest.mark.parametrize("world,dtype,mode,pieces", [(2, "fp32", "graph", 2), (3, "fp16", "graph", 4),
                                                    (2, "fp32", "graph_sharded", 0),
                                                    (3, "fp32", "graph_fused", 0),
                                                    (2, "fp16", "graph_push", 0)])
def test_ipc_cuda_graph_replay(orc, world, dtype, mode, pieces):
    """A captured CUDA graph of one multi-process step, replayed for steps
    1..3: device-resident barrier epochs advance on every replay, results
    stay bit-exact (pipelined schedule and sharded step)."""
    res = _run(world, dtype, "twoshot", steps=4, mode=mode, pieces=pieces)
    assert all(r[1] == "ok" for r in res), res
    shapes = synth.mlp_shapes()
    w = synth.params(shapes)
    v = [np.zeros_like(x) for x in w]
    for s in range(4):
        orc.step(synth.grads(shapes, workers=world, step=s), w, v, 0.1, 0.9, dtype)
    want_w = np.concatenate(w).view(np.uint32)
    for r in res:
        assert np.array_equal(np.frombuffer(r[2], np.uint32), want_w), f"rank {r[0]} w"


@pytest.mark.slow
@pytest.mark.parametrize("world,dtype,algo,mode,pieces", [(8, "fp32", "twoshot", "same", 0),
                                                        (8, "fp16", "twoshot", "same", 3),
                                                        (8, "fp16", "twoshot", "push", 0),
                                                        (4, "fp32", "oneshot", "fused", 0),
                                                        (5, "fp32", "twoshot", "sharded", 0)])
def test_ipc_many_ranks(orc, world, dtype, algo, mode, pieces):
    """4, 5 and 8 real processes (one GPU, time-sliced): every per-CTA
    barrier cell of an 8-rank signal pad in use, the N = 8 kernel
    instantiations across real IPC mappings; bit-exact w on every rank."""
    res = _run(world, dtype, algo, mode=mode, pieces=pieces)
    assert all(r[1] == "ok" for r in res), res
    shapes = synth.mlp_shapes()
    w = synth.params(shapes)
    v = [np.zeros_like(x) for x in w]
    for s in range(2):
        orc.step(synth.grads(shapes, workers=world, step=s), w, v, 0.1, 0.9, dtype)
    for r in res:
        assert np.array_equal(np.frombuffer(r[2], np.uint32), np.concatenate(w).view(np.uint32)), r[0]


@pytest.mark.slow
@pytest.mark.parametrize("dtype,mode,pieces", [("fp32", "r50:same", 4), ("fp16", "r50:push", 0)])
def test_ipc_r50_full_size(orc, dtype, mode, pieces):
    """The bench's workload at N = 2 across two real processes: the full
    ResNet-50 gradient set, pipelined (4 pieces, the default) and push-fused
    schedules, 2 steps; every rank's w and v bit-exact with the oracle
    (compared by SHA-256 of all 25.6M elements)."""
    import hashlib
    res = _run(2, dtype, "twoshot", mode=mode, pieces=pieces)
    assert all(r[1] == "ok" for r in res), res
    shapes = synth.resnet50_shapes()
    w = synth.params(shapes)
    v = [np.zeros_like(x) for x in w]
    for s in range(2):
        orc.step(synth.grads(shapes, workers=2, step=s), w, v, 0.1, 0.9, dtype)
    hw = hashlib.sha256(np.concatenate(w).tobytes()).hexdigest()
    hv = hashlib.sha256(np.concatenate(v).tobytes()).hexdigest()
    for r in res:
        assert r[2] == hw and r[3] == hv, f"rank {r[0]}"


@pytest.mark.slow
@pytest.mark.parametrize("world,dtype", [(3, "fp32"), (2, "fp16")])
def test_ipc_stress_random_schedules(orc, world, dtype):
    """60 steps across real processes with the schedule, algorithm and grid
    sizes redrawn every step (same draw on every rank): the per-CTA barrier
    epochs, buffer parities and inbox reuse stay paired; w and v bit-exact
    with 60 oracle steps on every rank."""
    steps = int(os.environ.get("CMN_STRESS_STEPS", "60"))     # longer soak runs: set CMN_STRESS_STEPS
    res = _run(world, dtype, "twoshot", steps=steps, mode="stress")
    assert all(r[1] == "ok" for r in res), res
    shapes = synth.mlp_shapes()
    w = synth.params(shapes)
    v = [np.zeros_like(x) for x in w]
    for s in range(steps):
        orc.step(synth.grads(shapes, workers=world, step=s), w, v, 0.1, 0.9, dtype)
    for r in res:
        assert np.array_equal(np.frombuffer(r[2], np.uint32), np.concatenate(w).view(np.uint32)), r[0]
        assert np.array_equal(np.frombuffer(r[3], np.uint32), np.concatenate(v).view(np.uint32)), r[0]


def test_ipc_single_call_schedule_refuses_capture():
    res = _run(2, "fp32", "oneshot", mode="capture_unpipelined")
    assert all(r[1] == "error" and r[2] == "CMN_ERR_UNSUPPORTED" for r in res), res


@pytest.mark.parametrize("world,dtype,mode", [(2, "fp16", "fused"), (3, "fp32", "fused"),
                                              (2, "fp32", "push"), (3, "fp16", "push")])
def test_ipc_fused_allgather_update(orc, world, dtype, mode):
    res = _run(world, dtype, "twoshot", mode=mode)
    assert all(r[1] == "ok" for r in res), res
    shapes = synth.mlp_shapes()
    w = synth.params(shapes)
    v = [np.zeros_like(x) for x in w]
    for s in range(2):
        orc.step(synth.grads(shapes, workers=world, step=s), w, v, 0.1, 0.9, dtype)
    for r in res:
        assert np.array_equal(np.frombuffer(r[2], np.uint32), np.concatenate(w).view(np.uint32))
        assert np.array_equal(np.frombuffer(r[3], np.uint32), np.concatenate(v).view(np.uint32))


@pytest.mark.parametrize("world,dtype,pieces", [(2, "fp32", 3), (3, "fp16", 0)])
def test_ipc_step_adam(orc, world, dtype, pieces):
    """cmn_step_adam across processes (pipelined per-piece Adam, or
    all-reduce then update): every rank's w bit-exact with the oracle."""
    res = _run(world, dtype, "twoshot", mode="adam", pieces=pieces)
    assert all(r[1] == "ok" for r in res), res
    shapes = synth.mlp_shapes()
    sizes = [synth.numel(x) for x in shapes]
    off, L = orc.layout(sizes)
    w = synth.params(shapes)
    m = [np.zeros_like(x) for x in w]
    v = [np.zeros_like(x) for x in w]
    for s in range(2):
        g = synth.grads(shapes, workers=world, step=s)
        red = orc.reduce_tree([orc.pack(gw, off, L, dtype) for gw in g], dtype)
        orc.update_adam(red, dtype, world, 1e-3, 0.9, 0.999, 1e-8, s + 1, off, w, m, v)
    for r in res:
        assert np.array_equal(np.frombuffer(r[2], np.uint32), np.concatenate(w).view(np.uint32)), r[0]


@pytest.mark.parametrize("world,dtype,pieces", [(2, "fp32", 3), (3, "fp16", 0)])
def test_ipc_step_host_packed(orc, world, dtype, pieces):
    """cmn_step_host_packed across processes: pinned host gradients in,
    host parameters out (pipelined per piece, or around a serial step);
    bit-exact with the oracle on every rank, host copy == device params."""
    res = _run(world, dtype, "twoshot", mode="host", pieces=pieces)
    assert all(r[1] == "ok" for r in res), res
    shapes = synth.mlp_shapes()
    w = synth.params(shapes)
    v = [np.zeros_like(x) for x in w]
    for s in range(2):
        orc.step(synth.grads(shapes, workers=world, step=s), w, v, 0.1, 0.9, dtype)
    for r in res:
        assert np.array_equal(np.frombuffer(r[2], np.uint32), np.concatenate(w).view(np.uint32))
        assert np.array_equal(np.frombuffer(r[3], np.uint32), np.concatenate(v).view(np.uint32))


@pytest.mark.parametrize("world,dtype", [(2, "fp32"), (3, "fp16")])
def test_ipc_mixed_schedules_and_grids(orc, world, dtype):
    """Schedules (fused, pipelined, serial) and CTA counts (cmn_set_ctas)
    switched between steps: bit-exact with the oracle on every rank."""
    res = _run(world, dtype, "twoshot", steps=7, mode="mixed")
    assert all(r[1] == "ok" for r in res), res
    shapes = synth.mlp_shapes()
    w = synth.params(shapes)
    v = [np.zeros_like(x) for x in w]
    for s in range(7):
        orc.step(synth.grads(shapes, workers=world, step=s), w, v, 0.1, 0.9, dtype)
    for r in res:
        assert np.array_equal(np.frombuffer(r[2], np.uint32), np.concatenate(w).view(np.uint32))
        assert np.array_equal(np.frombuffer(r[3], np.uint32), np.concatenate(v).view(np.uint32))


@pytest.mark.parametrize("algo", ["nvls", "nccl"])
def test_ipc_collective_setup_outcome_agrees(algo):
    """cmn_set_algo(NVLS | NCCL) with 2 processes: both ranks end with the
    same status (on the one-GPU boxes: multicast refused / NCCL refusing two
    ranks on one device), and neither blocks."""
    res = _run(2, "fp32", algo, mode="setup_alt")
    assert len({r[1:] for r in res}) == 1, res


def test_ipc_reregistration(orc):
    """Re-registration between steps (structure may change
    per iteration) is a collective that drains peers before freeing the
    IPC-exported buffers; momentum restarts from zero."""
    res = _run(2, "fp32", "twoshot", mode="reregister")
    assert all(r[1] == "ok" for r in res), res
    shapes = synth.mlp_shapes()
    w = synth.params(shapes)
    v = [np.zeros_like(x) for x in w]
    orc.step(synth.grads(shapes, workers=2, step=0), w, v, 0.1, 0.9, "fp32")
    v = [np.zeros_like(x) for x in w]
    orc.step(synth.grads(shapes, workers=2, step=1), w, v, 0.1, 0.9, "fp32")
    for r in res:
        assert np.array_equal(np.frombuffer(r[2], np.uint32), np.concatenate(w).view(np.uint32))
        assert np.array_equal(np.frombuffer(r[3], np.uint32), np.concatenate(v).view(np.uint32))


@pytest.mark.parametrize("algo,pieces", [("oneshot", 0), ("twoshot", 0), ("oneshot", 2), ("twoshot", 3)])
def test_ipc_skipped_collective_times_out(algo, pieces):
    """Fault injection: rank 1 skips one step (every collective of it).
    Rank 0's call 2 pairs with rank 1's call 3 (same layout, same kinds: a
    skipped whole step is indistinguishable by design), and rank 0's last
    call then finds no peer: its spin-wait times out (3 s), the error
    surfaces as CMN_ERR_TIMEOUT, and -- every later kernel
    checks the device error word -- that failed call leaves rank 0's w and v
    bit-identical to what they were before it (serial and pipelined
    schedules, one-shot and two-shot)."""
    res = _run(2, "fp32", algo, steps=3, mode="skip", pieces=pieces)
    statuses = {r[0]: r[1:] for r in res}
    assert statuses[0][0] == "error" and statuses[0][1] == "CMN_ERR_TIMEOUT", res
    assert statuses[0][2] is True, "the timed-out call modified rank 0's w / v"


def test_ipc_piece_mismatch_detected_outputs_untouched():
    """Ranks that cut the step into different pieces (rank 0 one collective
    over the whole model, rank 1 the pipelined schedule's first piece) issue
    all-reduces over different packed ranges at the same epoch: the
    barrier's call tag (range hash) turns that into CMN_ERR_MISMATCH instead
    of reducing unrelated ranges, and neither rank's w or v changes."""
    res = _run(2, "fp32", "twoshot", steps=1, mode="piece_mismatch", pieces=1)
    assert all(r[1] == "error" for r in res), res
    assert any(r[2] == "CMN_ERR_MISMATCH" for r in res), res
    assert all(r[2] in ("CMN_ERR_MISMATCH", "CMN_ERR_TIMEOUT") for r in res), res
    assert all(r[3] is True for r in res), res


@pytest.mark.parametrize("mode,dtype", [("slow_peer", "fp32"), ("slow_peer_graph", "fp16")])
def test_ipc_oneshot_pipelined_slow_peer(orc, mode, dtype):
    """Advisor finding (pipelined step, one-shot all-reduce): rank 1's
    one-shot CTAs stall 20 ms after the start barrier, so rank 0 finishes
    its all-reduce of the last piece and, with an even piece count, packs
    the next step's gradients into the very region rank 1 has not read yet.
    The last piece's end barrier must hold rank 0 back: w and v stay
    bit-exact with the oracle on both ranks, eagerly and replayed from a
    captured CUDA graph (same buffers every replay)."""
    res = _run(2, dtype, "oneshot", steps=3, mode=mode, pieces=4)
    assert all(r[1] == "ok" for r in res), res
    shapes = synth.mlp_shapes()
    w = synth.params(shapes)
    v = [np.zeros_like(x) for x in w]
    for s in range(3):
        orc.step(synth.grads(shapes, workers=2, step=s), w, v, 0.1, 0.9, dtype)
    for r in res:
        assert np.array_equal(np.frombuffer(r[2], np.uint32), np.concatenate(w).view(np.uint32)), r[0]


def test_ipc_structure_mismatch_detected():
    res = _run(2, "fp32", "oneshot", mode="mismatch")
    assert [r[1] for r in res] == ["error", "error"]
    assert all(r[2] == "CMN_ERR_MISMATCH" for r in res)
