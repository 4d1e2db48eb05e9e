"""Multi-process host logic of the N > 1 path on CPU (gloo, world_size 2):
the bootstrap allgather through torch.distributed, the registration-time
structure check ("model structures are identical between workers merely in
a single iteration") returning CMN_ERR_MISMATCH on every
rank when they differ, and identical layout / chunk plans on every rank."""
import os
import socket

import pytest
import torch.multiprocessing as mp

import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, q):
    import torch.distributed as dist

    from paper_1908_00213_b200 import cmn
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shapes = synth.mlp_shapes()
        if mode == "mismatch" and rank == 1:
            shapes = shapes[:-1] + [(11,)]            # one rank's model differs
        if mode == "transposed" and rank == 1:
            shapes = [(784, 100)] + shapes[1:]          # same numel, other structure
        off, L, h = cmn.plan_layout(shapes)
        st = cmn.bootstrap_verify(rank, world, h)
        s, e = cmn.plan_chunks(L, world)
        q.put((rank, st, off, L, s, e))
    finally:
        dist.destroy_process_group()


def _fd_worker(rank, world, port, path, q):
    import torch.distributed as dist

    from paper_1908_00213_b200 import cmn
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fd = os.open(path, os.O_RDONLY) if rank == 0 else -1
        got = cmn.share_fd(rank, world, fd)
        q.put((rank, os.pread(got, 64, 0).decode()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_share_fd_scm_rights(tmp_path, world):
    """The NVLS multicast-handle hand-off: rank 0's open file descriptor
    reaches every rank through an abstract Unix socket (SCM_RIGHTS) whose
    name travels through the bootstrap allgather."""
    from paper_1908_00213_b200 import build
    build.build()
    path = tmp_path / "payload"
    path.write_text("multicast-handle-stand-in")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_fd_worker, args=(r, world, port, str(path), q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[1] == "multicast-handle-stand-in" for r in res)


def _run(mode, world=2):
    from paper_1908_00213_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res)


@pytest.mark.parametrize("world", [2, 3])
def test_bootstrap_agrees(world):
    res = _run("same", world)
    assert all(r[1] == 0 for r in res)
    assert all(r[2:] == res[0][2:] for r in res)


@pytest.mark.parametrize("mode", ["mismatch", "transposed"])
def test_bootstrap_mismatch_on_every_rank(mode):
    res = _run(mode)
    assert [r[1] for r in res] == [5, 5]      # CMN_ERR_MISMATCH on both ranks


def _agree_worker(rank, world, port, q):
    import sys
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        # rank 1's budget ran out, the others' did not: nobody continues
        out = [bench.all_ranks_agree(rank != 1), bench.all_ranks_agree(True), bench.all_ranks_agree(False)]
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_bench_budget_decisions_are_collective(world):
    """bench.py's autotune / sweep budget stop is decided collectively (MIN
    over ranks): with one rank out of budget every rank stops, so no rank
    issues a collective its peers skip (the divergence that hung the
    time-sliced N = 8 run once)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_agree_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)])
    for p in ps:
        p.join(timeout=60)
    assert all(r[1] == [False, True, False] for r in res), res


def _probe_worker(rank, world, port, q):
    import sys
    import types
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        args = types.SimpleNamespace(dtype="fp32")
        res, adopted = bench.nvls_probe(args, rank, world, 0, timeout_s=240)
        q.put((rank, res, adopted))
    finally:
        dist.destroy_process_group()


def test_bench_nvls_probe_failure_is_contained_and_collective():
    """bench.py's isolated NVLS probe on a host without a GPU: every rank's
    child process fails (no CUDA device), the parent ranks survive, report
    why, and agree collectively not to adopt NVLS (the host side of the
    probe that shields an N > 1 run from a fault in the multimem kernel)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_probe_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(2)], key=lambda r: r[0])
    for p in ps:
        p.join(timeout=60)
    for rank, r, adopted in res:
        assert adopted is False
        assert r["probe"].startswith("child process") and "unavailable" in r and r["probe_s"] > 0
