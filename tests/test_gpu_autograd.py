"""NEXT-2: a real autograd producer in front of the path.

* bn-equivalence (§6.1.1: "the gradient obtained through
  communication is equivalent to that in the batch size bn"): N simulated
  workers each backpropagate a mean loss over their b-sample shard; the
  all-reduced average (cmn_unpack_avg_grads) equals the single-process
  gradient of the concatenated bn batch up to fp32 summation order
  (SPEC.md:587 states 1e-10 in f64; the fp32 bound used here is
  |d| <= 1e-4 |g| + 1e-7).
* Define-by-Run dynamic structure: the model changes depth
  between iterations; MultiNodeOptimizer re-registers and keeps training.
* Overlap via backward hooks: bucket all-reduces launched
  from post-accumulate-grad hooks give bitwise the same parameters as the
  unbucketed step.
"""
import pytest
import torch

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


@pytest.fixture(scope="module")
def cmn(cmn_worlds):
    """Every test here runs in the simulated and in the emulated world
    (conftest.cmn_worlds: barriers live in one cooperative launch)."""
    return cmn_worlds


def mlp(depth=3, seed=0):
    torch.manual_seed(seed)
    dims = [784] + [100] * (depth - 1) + [10]
    layers = []
    for i in range(depth):
        layers.append(torch.nn.Linear(dims[i], dims[i + 1]))
        if i < depth - 1:
            layers.append(torch.nn.ReLU())
    return torch.nn.Sequential(*layers).to(DEV)


def data(n, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    x = torch.randn(n, 784, generator=g)
    y = torch.randint(0, 10, (n,), generator=g)
    return x.to(DEV), y.to(DEV)


def worker_grads(model, x, y, N):
    """Each worker's gradient of its shard's mean loss (detached copies)."""
    b = x.shape[0] // N
    out = []
    for i in range(N):
        model.zero_grad(set_to_none=True)
        loss = torch.nn.functional.cross_entropy(model(x[i * b:(i + 1) * b]), y[i * b:(i + 1) * b])
        loss.backward()
        out.append([p.grad.detach().clone() for p in model.parameters()])
    return out


@pytest.mark.parametrize("N,dtype", [(2, "fp32"), (4, "fp32"), (8, "fp32"), (8, "fp16")])
def test_bn_equivalence(cmn, N, dtype):
    model = mlp()
    x, y = data(32 * N, seed=N)
    gw = worker_grads(model, x, y, N)
    model.zero_grad(set_to_none=True)
    torch.nn.functional.cross_entropy(model(x), y).backward()
    full = [p.grad.detach().clone() for p in model.parameters()]
    comm = cmn.Comm.simulated_world(N)
    try:
        params = list(model.parameters())
        comm.register_params([p.data for p in params])
        comm.allreduce_grads(gw, dtype)
        avg = [torch.empty_like(p) for p in params]
        comm.unpack_avg_grads(avg)
        torch.cuda.synchronize()
        rtol = 1e-4 if dtype == "fp32" else 2e-3
        for a, f in zip(avg, full):
            assert torch.all((a - f).abs() <= rtol * f.abs() + (1e-7 if dtype == "fp32" else 3e-5)), \
                float((a - f).abs().max())
    finally:
        comm.finalize()


def test_multi_node_optimizer_trains_and_matches_large_batch(cmn):
    """N = 4 workers x b = 16 with momentum SGD for 5 steps vs one process on
    the bn = 64 batch with torch.optim.SGD(momentum, dampening=0): parameters
    agree to fp32 summation-order tolerance, and the loss decreases."""
    from paper_1908_00213_b200.optim import MultiNodeOptimizer
    N = 4
    model = mlp(seed=3)
    ref = mlp(seed=3)
    comm = cmn.Comm.simulated_world(N)
    try:
        params = [p.data for p in model.parameters()]
        comm.register_params(params)
        opt_ref = torch.optim.SGD(ref.parameters(), lr=0.05, momentum=0.9)
        losses = []
        for it in range(5):
            x, y = data(16 * N, seed=100 + it)
            gw = worker_grads(model, x, y, N)
            comm.step(gw, "fp32", 0.05, 0.9)
            opt_ref.zero_grad()
            loss = torch.nn.functional.cross_entropy(ref(x), y)
            loss.backward()
            opt_ref.step()
            losses.append(float(loss.detach()))
        torch.cuda.synchronize()
        for p, q in zip(model.parameters(), ref.parameters()):
            assert torch.allclose(p, q, rtol=1e-4, atol=1e-6), float((p - q).abs().max())
        assert losses[-1] < losses[0]
    finally:
        comm.finalize()


def test_dynamic_structure_reregisters(cmn):
    """Depth alternates 3 -> 4 -> 3 across iterations (same on every worker);
    MultiNodeOptimizer re-registers on each change and the step matches
    plain momentum SGD on the averaged gradient of that iteration."""
    from paper_1908_00213_b200.optim import MultiNodeOptimizer
    comm = cmn.Comm.init(0, 1, 0)
    try:
        models = {3: mlp(3, seed=5), 4: mlp(4, seed=6)}
        opt = None
        for it, depth in enumerate([3, 4, 3, 3]):
            m = models[depth]
            x, y = data(32, seed=200 + it)
            m.zero_grad(set_to_none=True)
            torch.nn.functional.cross_entropy(m(x), y).backward()
            before = [p.detach().clone() for p in m.parameters()]
            grads = [p.grad.detach().clone() for p in m.parameters()]
            if opt is None:
                opt = MultiNodeOptimizer(list(m.parameters()), comm, lr=0.1, momentum=0.0)
                changed = True
            else:
                changed = opt.maybe_reregister(m.parameters())
            opt.step()
            torch.cuda.synchronize()
            assert changed == (it in (0, 1, 2))
            for p, b, g in zip(m.parameters(), before, grads):
                # mu = 0: w' = RN(w - 0.1 g) (one fma); torch's reference rounds twice
                assert torch.allclose(p.detach(), b - 0.1 * g, rtol=1e-6, atol=1e-8)
        assert opt.registrations == 3
    finally:
        comm.finalize()


def test_backward_hook_overlap_bitwise(cmn):
    """Bucket all-reduces launched from backward hooks (comm stream) give the
    same parameters, bit for bit, as the unbucketed cmn_step (N = 1 comm:
    the path is pack -> identity -> update per bucket)."""
    from paper_1908_00213_b200.optim import MultiNodeOptimizer
    results = []
    for bucket_bytes in (None, 64 << 10):
        model = mlp(seed=9)
        comm = cmn.Comm.init(0, 1, 0)
        try:
            opt = MultiNodeOptimizer(list(model.parameters()), comm, lr=0.05, momentum=0.9,
                                     bucket_bytes=bucket_bytes)
            for it in range(3):
                x, y = data(64, seed=300 + it)
                opt.zero_grad()
                torch.nn.functional.cross_entropy(model(x), y).backward()
                opt.step()
            torch.cuda.synchronize()
            if bucket_bytes:
                assert len(opt.buckets) > 1
            results.append(torch.cat([p.detach().reshape(-1) for p in model.parameters()]))
        finally:
            comm.finalize()
    assert torch.equal(results[0].view(torch.int32), results[1].view(torch.int32))


def test_multi_node_optimizer_adam_matches_large_batch(cmn):
    """The paper's Fig. 4 wraps Adam: N = 2 simulated workers through
    cmn_allreduce_grads + cmn_update_adam vs an fp64 Adam (Kingma & Ba's
    alpha_t form, eps added to sqrt(v) -- the form the library implements;
    torch.optim.Adam adds eps after the bias correction, a different
    optimizer for |g| near eps) driven by the single-process bn-batch
    gradient, 4 steps.  Adam's step is ~alpha*sign(g) where the averaged
    gradient nearly cancels, so such elements may flip between summation
    orders: 99.9 % must agree tightly, the rest within the 4-step bound."""
    N = 2
    model = mlp(seed=13)
    ref = mlp(seed=13)
    a, b1, b2, eps = 1e-3, 0.9, 0.999, 1e-8
    comm = cmn.Comm.simulated_world(N)
    try:
        comm.register_params([p.data for p in model.parameters()])
        w64 = [q.detach().double().clone() for q in ref.parameters()]
        m64 = [torch.zeros_like(x) for x in w64]
        v64 = [torch.zeros_like(x) for x in w64]
        for it in range(4):
            x, y = data(16 * N, seed=400 + it)
            gw = worker_grads(model, x, y, N)
            comm.allreduce_grads(gw, "fp32")
            comm.update_adam(a, b1, b2, eps, it + 1)
            with torch.no_grad():
                for q, w_ in zip(ref.parameters(), w64):
                    q.copy_(w_)
            ref.zero_grad()
            torch.nn.functional.cross_entropy(ref(x), y).backward()
            t = it + 1
            at = a * (1 - b2 ** t) ** 0.5 / (1 - b1 ** t)
            for q, w_, m_, v_ in zip(ref.parameters(), w64, m64, v64):
                g = q.grad.double()
                m_.mul_(b1).add_((1 - b1) * g)
                v_.mul_(b2).add_((1 - b2) * g * g)
                w_.sub_(at * m_ / (v_.sqrt() + eps))
        torch.cuda.synchronize()
        total, close = 0, 0
        for p, w_ in zip(model.parameters(), w64):
            d = (p.detach().double() - w_).abs()
            ok = d <= 1e-4 * w_.abs() + 2e-6
            total += d.numel()
            close += int(ok.sum())
            assert float(d.max()) <= 4 * a * 1.01
        assert close >= 0.999 * total, (close, total)
    finally:
        comm.finalize()


# ------------------------------------------------ oracle parity

def _host(gw):
    return [[g.detach().reshape(-1).cpu().numpy().copy() for g in w] for w in gw]


@pytest.mark.parametrize("N,dtype", [(2, "fp32"), (4, "fp16"), (8, "fp32"), (8, "fp16")])
def test_autograd_gradients_oracle_parity_simulated(cmn, orc, N, dtype):
    """NEXT-2 against the oracle: N simulated workers each backpropagate
    their own shard through the real model (torch autograd, the producer in
    front of the path); those per-worker gradients go through cmn_step and,
    as the same arrays, through oracle.step.  w and v must agree bitwise
    after every one of 4 steps (the next step's gradients are taken at the
    updated parameters, so the trajectory is pinned step by step)."""
    import numpy as np
    model = mlp(seed=21)
    params = list(model.parameters())
    w_o = [p.detach().reshape(-1).cpu().numpy().copy() for p in params]
    v_o = [np.zeros_like(x) for x in w_o]
    comm = cmn.Comm.simulated_world(N)
    try:
        comm.register_params([p.data for p in params])
        for it in range(4):
            x, y = data(8 * N, seed=500 + it)
            gw = worker_grads(model, x, y, N)
            gh = _host(gw)
            comm.step(gw, dtype, 0.05, 0.9)
            torch.cuda.synchronize()
            orc.step(gh, w_o, v_o, 0.05, 0.9, dtype)
            for t, p in enumerate(params):
                got_w = p.detach().reshape(-1).cpu().numpy()
                got_v = comm.momentum(t).reshape(-1).cpu().numpy()
                assert np.array_equal(got_w.view(np.uint32), w_o[t].view(np.uint32)), f"step {it} w[{t}]"
                assert np.array_equal(got_v.view(np.uint32), v_o[t].view(np.uint32)), f"step {it} v[{t}]"
    finally:
        comm.finalize()


def _mno_worker(rank, world, port, q, depths, bucket_bytes, dtype):
    import os

    import numpy as np
    import torch.distributed as dist

    from paper_1908_00213_b200 import cmn as cm
    from paper_1908_00213_b200.optim import MultiNodeOptimizer
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    global DEV
    try:
        dev = rank % torch.cuda.device_count()          # one GPU per rank
        DEV = f"cuda:{dev}"
        torch.cuda.set_device(dev)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        comm = cm.Comm.init(rank, world, dev, dist.group.WORLD)
        comm.set_timeout(60000)
        models = {d: mlp(d, seed=40 + d) for d in sorted(set(depths))}   # same init on every rank
        opt = None
        log = []
        for it, d in enumerate(depths):
            m = models[d]
            x, y = data(16, seed=1000 * rank + it)                        # this rank's own batch
            if opt is None:
                opt = MultiNodeOptimizer(list(m.parameters()), comm, lr=0.05, momentum=0.9, dtype=dtype,
                                         bucket_bytes=bucket_bytes)
            else:
                opt.maybe_reregister(m.parameters())   # collective when the structure changed
            opt.zero_grad()
            torch.nn.functional.cross_entropy(m(x), y).backward()
            grads = [p.grad.detach().reshape(-1).cpu().numpy().tobytes() for p in m.parameters()]
            opt.step()
            torch.cuda.synchronize()
            log.append((d, grads))
        final = {d: [p.detach().reshape(-1).cpu().numpy().tobytes() for p in m.parameters()]
                 for d, m in models.items()}
        mom = [comm.momentum(t).reshape(-1).cpu().numpy().tobytes() for t in range(len(opt.params))]
        q.put((rank, "ok", log, final, mom, opt.registrations))
        dist.barrier()
        comm.finalize()
    except Exception as e:  # noqa: BLE001
        q.put((rank, "exc", repr(e)))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("world,bucket_bytes,dtype", [(2, None, "fp32"), (3, None, "fp16"),
                                                      (2, 64 << 10, "fp32")])
def test_multi_node_optimizer_processes_oracle_parity(cmn, orc, world, bucket_bytes, dtype):
    """MultiNodeOptimizer across 2-3 real processes, one per GPU (CUDA-IPC barriers live),
    each rank backpropagating its own batch, the model's depth changing
    3 -> 3 -> 4 -> 4 -> 3 on every rank in the same iterations (PAPER.md:
    493-501, Define-by-Run; each change is a collective re-registration
    that resets momentum, reading R7), with and without backward-hook
    buckets.  The oracle replays the run from the gradients every rank
    produced: per iteration oracle.step over the N ranks' gradients of the
    registered model, v zeroed at each re-registration.  Every rank's final
    parameters of both models and its momentum must equal the oracle's
    bitwise.  One GPU per rank (conftest.require_gpus_for_ranks)."""
    import socket

    import numpy as np
    import torch.multiprocessing as mp

    from conftest import require_gpus_for_ranks
    require_gpus_for_ranks(world)
    depths = [3, 3, 4, 4, 3]
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_mno_worker, args=(r, world, port, q, depths, bucket_bytes, dtype))
          for r in range(world)]
    for p in ps:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda r: r[0])
    for p in ps:
        p.join(timeout=120)
    assert all(r[1] == "ok" for r in res), res
    assert all(r[5] == 3 for r in res)                       # registrations: 3, 4, 3
    # the oracle's replay
    init = {d: [p.detach().reshape(-1).cpu().numpy().copy() for p in mlp(d, seed=40 + d).parameters()]
            for d in sorted(set(depths))}
    w_o = {d: [x.copy() for x in init[d]] for d in init}
    v_o, cur = None, None
    for it, d in enumerate(depths):
        if d != cur:
            v_o = [np.zeros_like(x) for x in w_o[d]]
            cur = d
        g = [[np.frombuffer(b, np.float32).copy() for b in res[r][2][it][1]] for r in range(world)]
        assert all(res[r][2][it][0] == d for r in range(world))
        orc.step(g, w_o[d], v_o, 0.05, 0.9, dtype)
    for r in res:
        for d in w_o:
            for t, b in enumerate(r[3][d]):
                assert np.frombuffer(b, np.uint32).tobytes() == w_o[d][t].tobytes(), f"rank {r[0]} depth {d} w[{t}]"
        for t, b in enumerate(r[4]):
            assert b == v_o[t].tobytes(), f"rank {r[0]} v[{t}]"


def test_bucketed_reregistration_and_accumulation_guards(cmn):
    """Advisor findings on the hook state: (1) re-registering inside step()
    after a backward whose hooks launched buckets under the old plan must
    not leave stale bucket indices (the step completes and equals the
    unbucketed optimizer bitwise); (2) a second backward before step()
    raises instead of all-reducing a partial gradient, while no_sync()
    accumulation gives the unbucketed result; (3) Adam with buckets is
    refused."""
    from paper_1908_00213_b200.optim import MultiNodeOptimizer
    out = []
    for bucket_bytes in (None, 32 << 10):
        models = {3: mlp(3, seed=61), 4: mlp(4, seed=62)}
        comm = cmn.Comm.init(0, 1, 0)
        try:
            opt = MultiNodeOptimizer(list(models[3].parameters()), comm, lr=0.05, momentum=0.9,
                                     bucket_bytes=bucket_bytes)
            reg = 3
            for it, d in enumerate([3, 3, 4, 3]):
                m = models[d]
                if d != reg:
                    # a backward through the still-registered model first: its
                    # hooks launch bucket all-reduces under the old plan, then
                    # step() re-registers (the stale-index case)
                    for p in models[reg].parameters():
                        p.grad = None
                    x, y = data(16, seed=800 + it)
                    torch.nn.functional.cross_entropy(models[reg](x), y).backward()
                    reg = d
                for p in m.parameters():
                    p.grad = None
                with opt.no_sync():                        # accumulation micro-batch
                    x, y = data(16, seed=700 + 2 * it)
                    torch.nn.functional.cross_entropy(m(x), y).backward()
                x, y = data(16, seed=701 + 2 * it)
                torch.nn.functional.cross_entropy(m(x), y).backward()
                opt.step(m.parameters())                    # re-registers when d changed
            torch.cuda.synchronize()
            out.append(torch.cat([p.detach().reshape(-1) for d in (3, 4) for p in models[d].parameters()]))
            if bucket_bytes:
                m = models[3]
                x, y = data(16, seed=999)
                with pytest.raises(RuntimeError):
                    for _ in range(2):                      # second backward before step()
                        torch.nn.functional.cross_entropy(m(x), y).backward()
        finally:
            comm.finalize()
    assert torch.equal(out[0].view(torch.int32), out[1].view(torch.int32))
    comm = cmn.Comm.init(0, 1, 0)
    try:
        with pytest.raises(ValueError):
            MultiNodeOptimizer(list(mlp(3).parameters()), comm, optimizer="adam", bucket_bytes=1 << 20)
    finally:
        comm.finalize()


def test_binding_refuses_wrong_dtype_and_device(cmn):
    """Advisor finding: pointers of non-fp32, CPU or other-device tensors
    never reach the kernels (CMN_ERR_INVALID_ARG from the binding)."""
    comm = cmn.Comm.init(0, 1, 0)
    try:
        with pytest.raises(cmn.CmnError) as e:
            comm.register_params([torch.zeros(64, dtype=torch.float16, device=DEV)])
        assert e.value.status_name == "CMN_ERR_INVALID_ARG"
        with pytest.raises(cmn.CmnError):
            comm.register_params([torch.zeros(64)])          # CPU tensor
        w = [torch.zeros(64, device=DEV)]
        comm.register_params(w)
        with pytest.raises(cmn.CmnError):
            comm.step([torch.zeros(64, dtype=torch.bfloat16, device=DEV)], "fp32", 0.1, 0.9)
        with pytest.raises(cmn.CmnError):
            comm.step([torch.zeros(64)], "fp32", 0.1, 0.9)
    finally:
        comm.finalize()
