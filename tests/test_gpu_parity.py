"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded synthetic inputs, element by element.

Bar: the pack/unpack index mapping is bit-exact; the
hand-written fp32 and fp16 all-reduce + update are bit-exact too (same tree
order, same IEEE rounding, same explicit fma), and additionally inside the
north-star tolerance gate |a - abar| <= 1e-5 m (fp32) / 2e-3 m + 2^-24
(fp16) against the exact fp64 average.  NaNs are compared by position.

Simulated-N mode runs the same all-reduce kernels as the multi-process path
(N buffers on one device, one launch per simulated rank)."""
import numpy as np
import pytest
import torch

import synth
from conftest import single_rank_only

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


@pytest.fixture(scope="module")
def cmn(cmn_worlds):
    """Every test here runs in the simulated and in the emulated world
    (conftest.cmn_worlds: barriers live in one cooperative launch)."""
    return cmn_worlds


def _bits(x: np.ndarray) -> np.ndarray:
    return x.view(np.uint32) if x.dtype == np.float32 else x.view(np.uint16)


def assert_bitwise(got: np.ndarray, want: np.ndarray, what: str):
    assert got.shape == want.shape, what
    if got.dtype == np.float32:
        gn, wn = np.isnan(got), np.isnan(want)
    else:  # fp16 bits
        gn = ((got & 0x7C00) == 0x7C00) & ((got & 0x3FF) != 0)
        wn = ((want & 0x7C00) == 0x7C00) & ((want & 0x3FF) != 0)
    assert np.array_equal(gn, wn), f"{what}: NaN positions differ"
    ok = _bits(got)[~gn] == _bits(want)[~wn]
    if not ok.all():
        idx = np.flatnonzero(~gn)[np.flatnonzero(~ok)[:5]]
        raise AssertionError(f"{what}: {np.count_nonzero(~ok)} elements differ, e.g. at {idx}: "
                             f"got {got[idx]} want {want[idx]}")


def to_dev(arrs):
    return [torch.from_numpy(a.copy()).to(DEV) for a in arrs]


def run_gpu(cmn, shapes, N, dtype, algo, grads_by_step, params0, lr, mu, capture=True):
    comm = cmn.Comm.simulated_world(N)
    try:
        w = to_dev(params0)
        comm.register_params(w)
        comm.set_algo(algo)
        off, L = comm.layout()
        out = []
        tdt = torch.float32 if dtype == "fp32" else torch.int16
        for g in grads_by_step:
            gd = [to_dev(gw) for gw in g]
            comm.allreduce_grads(gd, dtype)
            rec = {}
            if capture:
                rec["packed"] = []
                rec["reduced"] = []
                for r in range(N):
                    p = torch.empty(L, dtype=tdt, device=DEV)
                    comm.copy_packed(r, p)
                    rec["packed"].append(p)
                    q = torch.empty(L, dtype=tdt, device=DEV)
                    comm.copy_reduced(r, q)
                    rec["reduced"].append(q)
            comm.update_momentum_sgd(lr, mu)
            torch.cuda.synchronize()
            rec = {k: [x.cpu().numpy() for x in v] for k, v in rec.items()}
            if dtype == "fp16":
                rec = {k: [x.view(np.uint16) for x in v] for k, v in rec.items()}
            rec["w"] = [x.cpu().numpy().reshape(-1) for x in w]
            rec["v"] = [comm.momentum(t).cpu().numpy().reshape(-1) for t in range(len(w))]
            out.append(rec)
        return out, off, L
    finally:
        comm.finalize()


def run_oracle(orc, shapes, N, dtype, grads_by_step, params0, lr, mu):
    w = [p.copy() for p in params0]
    v = [np.zeros_like(p) for p in params0]
    sizes = [synth.numel(s) for s in shapes]
    off, L = orc.layout(sizes)
    out = []
    for g in grads_by_step:
        packed = [orc.pack(gw, off, L, dtype) for gw in g]
        red = orc.reduce_tree(packed, dtype)
        orc.update_momentum_sgd(red, dtype, N, lr, mu, off, w, v)
        out.append({"packed": packed, "reduced": red, "w": [x.copy() for x in w],
                    "v": [x.copy() for x in v]})
    return out, off, L


def compare(gpu, ora, N, check_buffers=True):
    for s, (g, o) in enumerate(zip(gpu, ora)):
        if check_buffers:
            for r in range(N):
                assert_bitwise(g["packed"][r], o["packed"][r], f"step {s} packed rank {r}")
                assert_bitwise(g["reduced"][r], o["reduced"], f"step {s} reduced rank {r}")
        for t in range(len(o["w"])):
            assert_bitwise(g["w"][t], o["w"][t], f"step {s} w[{t}]")
            assert_bitwise(g["v"][t], o["v"][t], f"step {s} v[{t}]")


RAGGED = [(1,), (3,), (4097,), (8191,), (100, 100), (65,), (2, 3, 5), (12289,), (7,)]


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("dtype", ["fp32", "fp16"])
@pytest.mark.parametrize("algo", ["oneshot", "twoshot"])
def test_mlp_parity_bitexact(cmn, orc, N, dtype, algo):
    shapes = synth.mlp_shapes()
    grads = [synth.grads(shapes, workers=N, step=s) for s in range(2)]
    params0 = synth.params(shapes)
    gpu, goff, gL = run_gpu(cmn, shapes, N, dtype, algo, grads, params0, 0.1, 0.9)
    ora, ooff, oL = run_oracle(orc, shapes, N, dtype, grads, params0, 0.1, 0.9)
    assert goff == list(ooff) and gL == oL
    compare(gpu, ora, N)


@pytest.mark.parametrize("N", [1, 2, 7, 8])
@pytest.mark.parametrize("dtype", ["fp32", "fp16"])
@pytest.mark.parametrize("algo", ["oneshot", "twoshot"])
def test_ragged_shapes_parity(cmn, orc, N, dtype, algo):
    shapes = RAGGED
    grads = [synth.grads(shapes, workers=N, step=s, seed=7) for s in range(3)]
    params0 = synth.params(shapes, seed=7)
    gpu, _, _ = run_gpu(cmn, shapes, N, dtype, algo, grads, params0, 0.05, 0.5)
    ora, _, _ = run_oracle(orc, shapes, N, dtype, grads, params0, 0.05, 0.5)
    compare(gpu, ora, N)


@pytest.mark.parametrize("value_set", ["integer", "identical", "edge"])
@pytest.mark.parametrize("dtype", ["fp32", "fp16"])
def test_value_sets_parity(cmn, orc, value_set, dtype):
    shapes = synth.mlp_shapes()
    N = 4
    lr, mu = (2.0 ** -4, 2.0 ** -1) if value_set == "integer" else (0.1, 0.9)
    grads = [synth.grads(shapes, workers=N, step=s, value_set=value_set) for s in range(3)]
    params0 = synth.params(shapes, value_set="integer" if value_set == "integer" else "random")
    for algo in ("oneshot", "twoshot"):
        gpu, _, _ = run_gpu(cmn, shapes, N, dtype, algo, grads, params0, lr, mu)
        ora, _, _ = run_oracle(orc, shapes, N, dtype, grads, params0, lr, mu)
        compare(gpu, ora, N)


@pytest.mark.parametrize("dtype", ["fp32", "fp16"])
def test_tolerance_gate_vs_exact(cmn, orc, dtype):
    """North-star gate on the averaged gradient: unpack_avg vs fp64 exact."""
    shapes = synth.resnet50_shapes()[:20]
    N = 8
    g = synth.grads(shapes, workers=N)
    comm = cmn.Comm.simulated_world(N)
    try:
        w = to_dev(synth.params(shapes))
        comm.register_params(w)
        comm.allreduce_grads([to_dev(gw) for gw in g], dtype)
        out = [torch.empty_like(x) for x in w]
        comm.unpack_avg_grads(out)
        torch.cuda.synchronize()
        off, L = comm.layout()
        p32 = [orc.pack(gw, off, L, "fp32") for gw in g]
        avg, mag = orc.exact_avg(p32)
        for t, o in enumerate(out):
            a = o.cpu().numpy().reshape(-1).astype(np.float64)
            n = a.size
            ex, m = avg[off[t]: off[t] + n], mag[off[t]: off[t] + n]
            if dtype == "fp32":
                assert np.all(np.abs(a - ex) <= 1e-5 * m)
            else:
                assert np.all(np.abs(a - ex) <= 2e-3 * m + 2.0 ** -24)
    finally:
        comm.finalize()


def test_step_n1_direct_equals_unfused(cmn, orc):
    """cmn_step at N = 1 (no pack, the bench's kernel) == allreduce+update ==
    oracle, bitwise, for fp32 and fp16, over 3 steps."""
    single_rank_only(cmn)
    shapes = synth.mlp_shapes() + RAGGED
    for dtype in ("fp32", "fp16"):
        grads = [synth.grads(shapes, workers=1, step=s) for s in range(3)]
        params0 = synth.params(shapes)
        ora, _, _ = run_oracle(orc, shapes, 1, dtype, grads, params0, 0.1, 0.9)
        comm = cmn.Comm.init(0, 1, 0)
        try:
            w = to_dev(params0)
            comm.register_params(w)
            for s, g in enumerate(grads):
                comm.step(to_dev(g[0]), dtype, 0.1, 0.9)
                torch.cuda.synchronize()
                for t in range(len(w)):
                    assert_bitwise(w[t].cpu().numpy().reshape(-1), ora[s]["w"][t], f"w[{t}] step {s}")
                    assert_bitwise(comm.momentum(t).cpu().numpy().reshape(-1), ora[s]["v"][t], f"v[{t}]")
        finally:
            comm.finalize()


@pytest.mark.slow
@pytest.mark.parametrize("dtype", ["fp32", "fp16"])
def test_r50_full_size_n1_bench_config(cmn, orc, dtype):
    """BASELINE configs 2 / 3 at N = 1 in exactly the launch configuration
    bench.py times: parameters and gradients as views of one flat allocation
    each in the packed layout, a pre-marshalled pointer table, cmn_step on
    torch's current stream, 3 steps; all 25.6M elements of w and v vs the
    oracle after every step."""
    single_rank_only(cmn)
    shapes = synth.resnet50_shapes()
    sizes = [synth.numel(s) for s in shapes]
    params0 = synth.params(shapes)
    w_o = [p.copy() for p in params0]
    v_o = [np.zeros_like(p) for p in params0]
    off, L, _ = cmn.plan_layout(shapes)
    comm = cmn.Comm.init(0, 1, 0)
    try:
        flat_w = torch.empty(L, dtype=torch.float32, device=DEV)
        w = [flat_w[off[t]: off[t] + sizes[t]].view(shapes[t]) for t in range(len(shapes))]
        for t in range(len(w)):
            w[t].copy_(torch.from_numpy(params0[t]).view(shapes[t]))
        comm.register_params(w)
        flat_g = torch.empty(L, dtype=torch.float32, device=DEV)
        gv = [flat_g[off[t]: off[t] + sizes[t]] for t in range(len(shapes))]
        table = comm.prepare(gv)
        for step in range(3):
            g = synth.grads(shapes, workers=1, step=step)
            for t in range(len(gv)):
                gv[t].copy_(torch.from_numpy(g[0][t]))
            orc.step(g, w_o, v_o, 0.1, 0.9, dtype)
            comm.step(table, dtype, 0.1, 0.9)
            torch.cuda.synchronize()
            got_w = flat_w.cpu().numpy()
            for t in range(len(w)):
                assert_bitwise(got_w[off[t]: off[t] + sizes[t]].copy(), w_o[t], f"w[{t}] step {step}")
                assert_bitwise(comm.momentum(t).cpu().numpy().reshape(-1), v_o[t], f"v[{t}] step {step}")
    finally:
        comm.finalize()


@pytest.mark.slow
@pytest.mark.parametrize("dtype,algo", [("fp32", "twoshot"), ("fp16", "twoshot"), ("fp16", "oneshot")])
def test_r50_full_size_n8_simulated(cmn, orc, dtype, algo):
    """ResNet-50 gradient set, 8 simulated workers, full size: reduced buffer
    of every rank and the updated w, v, all elements, bit-exact."""
    shapes = synth.resnet50_shapes()
    N = 8
    grads = [synth.grads(shapes, workers=N)]
    params0 = synth.params(shapes)
    gpu, _, _ = run_gpu(cmn, shapes, N, dtype, algo, grads, params0, 0.1, 0.9)
    ora, _, _ = run_oracle(orc, shapes, N, dtype, grads, params0, 0.1, 0.9)
    compare(gpu, ora, N)


@pytest.mark.slow
@pytest.mark.parametrize("N,dtype,algo", [(2, "fp32", "oneshot"), (3, "fp16", "twoshot")])
def test_max_size_buffer_sampled(cmn, orc, N, dtype, algo):
    """The largest buffer of the config-5 sweep (1 GiB of fp32, one tensor of
    2^28 + 37 elements: ragged tail, pad, uneven two-shot chunks), allreduce
    + update at N simulated workers.  Every step of the method after the
    layout is elementwise, so the oracle run on a sample of element indices
    (both ends, chunk boundaries, 2^18 random) gives exactly the expected
    values there; the rest is checked to be finite and changed."""
    n = (1 << 28) + 37
    grads = [[synth.grad_tensor(n, 0, worker=i)] for i in range(N)]
    w0 = synth.param_tensor(n, 0)
    starts, ends = cmn.plan_chunks(-(-n // 64) * 64, N)
    rng = np.random.default_rng(5)
    edges = np.concatenate([np.arange(0, 4096), np.arange(n - 4096, n)] +
                           [np.arange(max(0, b - 64), min(n, b + 64)) for b in list(starts) + list(ends)])
    idx = np.unique(np.concatenate([edges, rng.integers(0, n, 1 << 18)]))
    comm = cmn.Comm.simulated_world(N)
    try:
        w = torch.from_numpy(w0).to(DEV)
        comm.register_params([w])
        comm.set_algo(algo)
        gd = [[torch.from_numpy(gw[0]).to(DEV)] for gw in grads]
        del grads[1:]
        comm.allreduce_grads(gd, dtype)
        comm.update_momentum_sgd(0.1, 0.9)
        torch.cuda.synchronize()
        del gd
        got_w = w.cpu().numpy()
        got_v = comm.momentum(0).cpu().numpy().reshape(-1)
    finally:
        comm.finalize()
    gs = [[synth.grad_tensor(n, 0, worker=i)[idx].copy()] for i in range(N)]
    ws, vs = [w0[idx].copy()], [np.zeros(len(idx), np.float32)]
    orc.step(gs, ws, vs, 0.1, 0.9, dtype)
    assert_bitwise(got_w[idx], ws[0], "w (sampled)")
    assert_bitwise(got_v[idx], vs[0], "v (sampled)")
    assert np.isfinite(got_w).all() and np.isfinite(got_v).all()
    assert np.count_nonzero(got_v == 0) < n // 1000     # every element was updated


@pytest.mark.parametrize("N,pieces,dtype", [(2, 2, "fp32"), (4, 3, "fp16"), (8, 4, "fp32"),
                                            (3, 7, "fp16"), (8, 16, "fp16")])
def test_pipelined_step_parity(cmn, orc, N, pieces, dtype):
    """cmn_step at N > 1 with the pipelined schedule (packs/updates on the
    caller stream, all-reduces on the communication stream, one collective
    per piece) == oracle, bitwise, over 3 steps (buffer parity reuse)."""
    shapes = synth.resnet50_shapes()[:50] + RAGGED
    grads = [synth.grads(shapes, workers=N, step=s) for s in range(3)]
    params0 = synth.params(shapes)
    ora, _, _ = run_oracle(orc, shapes, N, dtype, grads, params0, 0.1, 0.9)
    comm = cmn.Comm.simulated_world(N)
    try:
        w = to_dev(params0)
        comm.register_params(w)
        comm.set_pipeline(pieces)
        for s, g in enumerate(grads):
            comm.step(comm.prepare([to_dev(gw) for gw in g]), dtype, 0.1, 0.9)
            torch.cuda.synchronize()
            for t in range(len(w)):
                assert_bitwise(w[t].cpu().numpy().reshape(-1), ora[s]["w"][t], f"w[{t}] step {s}")
                assert_bitwise(comm.momentum(t).cpu().numpy().reshape(-1), ora[s]["v"][t], f"v[{t}]")
    finally:
        comm.finalize()


@pytest.mark.parametrize("N,dtype,ctas,mode", [(2, "fp32", (0, 0), "pull"), (3, "fp16", (0, 0), "pull"),
                                               (4, "fp16", (3, 1), "pull"), (8, "fp32", (0, 0), "pull"),
                                               (8, "fp32", (1024, 1024), "pull"),
                                               (2, "fp32", (0, 0), "push"), (3, "fp16", (0, 0), "push"),
                                               (4, "fp16", (3, 1), "push"), (8, "fp32", (0, 0), "push"),
                                               (8, "fp16", (1024, 1024), "push"), (5, "fp32", (7, 2), "push")])
def test_fused_allgather_update_parity(cmn, orc, N, dtype, ctas, mode):
    """Fused two-shot step (reduce-scatter -- pulled from packed buffers, or
    pushed by the fused pack kernel into the owners' inboxes -- then one
    kernel updating every parameter from the owners' reduced chunks) ==
    oracle bitwise, 3 steps; also the reduced chunks, pads included."""
    shapes = synth.resnet50_shapes()[:30] + RAGGED
    grads = [synth.grads(shapes, workers=N, step=s) for s in range(3)]
    params0 = synth.params(shapes)
    ora, _, _ = run_oracle(orc, shapes, N, dtype, grads, params0, 0.1, 0.9)
    comm = cmn.Comm.simulated_world(N)
    try:
        w = to_dev(params0)
        comm.register_params(w)
        comm.set_fused_update(mode)
        comm.set_ctas(*ctas)            # grid sizes never change results
        _, L = comm.layout()
        starts, ends = cmn.plan_chunks(L, N)
        tdt = torch.float32 if dtype == "fp32" else torch.int16
        for s, g in enumerate(grads):
            comm.step([to_dev(gw) for gw in g], dtype, 0.1, 0.9)
            torch.cuda.synchronize()
            for t in range(len(w)):
                assert_bitwise(w[t].cpu().numpy().reshape(-1), ora[s]["w"][t], f"w[{t}] step {s}")
                assert_bitwise(comm.momentum(t).cpu().numpy().reshape(-1), ora[s]["v"][t], f"v[{t}]")
            for r in range(N):          # each owner's reduced chunk (pads included)
                q = torch.empty(L, dtype=tdt, device=DEV)
                comm.copy_reduced(r, q)
                got = q.cpu().numpy()
                if dtype == "fp16":
                    got = got.view(np.uint16)
                a, b = starts[r], ends[r]
                assert_bitwise(got[a:b], ora[s]["reduced"][a:b], f"reduced chunk {r} step {s}")
    finally:
        comm.finalize()


@pytest.mark.parametrize("N,dtype,ctas", [(2, "fp32", (0, 0)), (3, "fp16", (0, 0)), (4, "fp32", (7, 2)),
                                          (8, "fp16", (0, 0)), (8, "fp32", (0, 1024))])
def test_sharded_update_parity(cmn, orc, N, dtype, ctas):
    """NEXT-4 (cmn_step_sharded): reduce-scatter, update of the own chunk,
    all-gather of parameters == oracle bitwise over 3 steps (w, and v, which
    the simulated ranks together update in full)."""
    shapes = synth.resnet50_shapes()[:30] + RAGGED
    grads = [synth.grads(shapes, workers=N, step=s) for s in range(3)]
    params0 = synth.params(shapes)
    ora, _, _ = run_oracle(orc, shapes, N, dtype, grads, params0, 0.1, 0.9)
    comm = cmn.Comm.simulated_world(N)
    try:
        w = to_dev(params0)
        comm.register_params(w)
        comm.set_ctas(*ctas)
        for s, g in enumerate(grads):
            comm.step_sharded([to_dev(gw) for gw in g], dtype, 0.1, 0.9)
            torch.cuda.synchronize()
            for t in range(len(w)):
                assert_bitwise(w[t].cpu().numpy().reshape(-1), ora[s]["w"][t], f"w[{t}] step {s}")
                assert_bitwise(comm.momentum(t).cpu().numpy().reshape(-1), ora[s]["v"][t], f"v[{t}]")
    finally:
        comm.finalize()


def test_buckets_bitwise_equal_unbucketed(cmn, orc):
    """Overlap reading R15: bucketed (reverse order, any size) == unbucketed."""
    shapes = synth.resnet50_shapes()[:40]
    N = 4
    grads = [synth.grads(shapes, workers=N, step=s) for s in range(2)]
    params0 = synth.params(shapes)
    ora, _, _ = run_oracle(orc, shapes, N, "fp16", grads, params0, 0.1, 0.9)
    for bucket_bytes in (0, 1 << 16, 1 << 20, 4 << 20):
        comm = cmn.Comm.simulated_world(N)
        try:
            w = to_dev(params0)
            comm.register_params(w)
            nb = comm.plan_buckets(bucket_bytes)
            ranges = [comm.get_bucket(b) for b in range(nb)]
            assert ranges[0][1] == len(shapes) and ranges[-1][0] == 0
            for s, g in enumerate(grads):
                gd = [to_dev(gw) for gw in g]
                for b in range(nb):
                    comm.allreduce_bucket(b, gd, "fp16")
                for b in range(nb):
                    comm.update_bucket(b, 0.1, 0.9)
                torch.cuda.synchronize()
                for t in range(len(w)):
                    assert_bitwise(w[t].cpu().numpy().reshape(-1), ora[s]["w"][t], f"w[{t}]")
        finally:
            comm.finalize()


def test_adam_parity(cmn, orc):
    shapes = synth.mlp_shapes() + RAGGED
    N = 2
    sizes = [synth.numel(s) for s in shapes]
    off, L = orc.layout(sizes)
    params0 = synth.params(shapes)
    w_o = [p.copy() for p in params0]
    m_o = [np.zeros_like(p) for p in params0]
    v_o = [np.zeros_like(p) for p in params0]
    comm = cmn.Comm.simulated_world(N)
    try:
        w = to_dev(params0)
        comm.register_params(w)
        for step in range(1, 4):
            g = synth.grads(shapes, workers=N, step=step)
            red = orc.reduce_tree([orc.pack(gw, off, L, "fp32") for gw in g], "fp32")
            orc.update_adam(red, "fp32", N, 1e-3, 0.9, 0.999, 1e-8, step, off, w_o, m_o, v_o)
            comm.allreduce_grads([to_dev(gw) for gw in g], "fp32")
            comm.update_adam(1e-3, 0.9, 0.999, 1e-8, step)
            torch.cuda.synchronize()
            for t in range(len(w)):
                m, v = comm.adam_state(t)
                assert_bitwise(w[t].cpu().numpy().reshape(-1), w_o[t], f"adam w[{t}]")
                assert_bitwise(m.cpu().numpy().reshape(-1), m_o[t], f"adam m[{t}]")
                assert_bitwise(v.cpu().numpy().reshape(-1), v_o[t], f"adam v[{t}]")
    finally:
        comm.finalize()


def test_step_host_e2e_parity(cmn, orc):
    shapes = synth.mlp_shapes()
    g = synth.grads(shapes, workers=1)
    params0 = synth.params(shapes)
    w_o = [p.copy() for p in params0]
    v_o = [np.zeros_like(p) for p in params0]
    orc.step(g, w_o, v_o, 0.1, 0.9, "fp16")
    comm = cmn.Comm.init(0, 1, 0)
    try:
        w = to_dev(params0)
        comm.register_params(w)
        hg = [torch.from_numpy(x.copy()).pin_memory() for x in g[0]]
        hw = [torch.empty(x.shape, dtype=torch.float32).pin_memory() for x in params0]
        comm.step_host(hg, hw, "fp16", 0.1, 0.9)
        torch.cuda.synchronize()
        for t in range(len(hw)):
            assert_bitwise(hw[t].numpy().reshape(-1), w_o[t], f"host w[{t}]")
    finally:
        comm.finalize()


@pytest.mark.parametrize("flat_params,pieces", [(True, None), (False, None), (True, "1"),
                                                (False, "7"), (True, "64")])
@pytest.mark.parametrize("dtype", ["fp32", "fp16"])
def test_step_host_packed_pipelined_parity(cmn, orc, monkeypatch, flat_params, pieces, dtype):
    """cmn_step_host_packed at N = 1 (pipelined over item ranges that cut
    through tensors, two copy streams) over 3 steps, params as one flat
    allocation ending at the last tensor (not at L) or as separate ones;
    default ramped pieces and CMN_E2E_PIECES equal pieces."""
    if pieces is not None:
        monkeypatch.setenv("CMN_E2E_PIECES", pieces)
    shapes = synth.resnet50_shapes()[:60]
    sizes = [synth.numel(s) for s in shapes]
    off, L = orc.layout(sizes)
    params0 = synth.params(shapes)
    w_o = [p.copy() for p in params0]
    v_o = [np.zeros_like(p) for p in params0]
    comm = cmn.Comm.init(0, 1, 0)
    try:
        if flat_params:
            flat = torch.zeros(off[len(sizes) - 1] + sizes[-1], dtype=torch.float32, device=DEV)
            w = [flat[off[t]: off[t] + sizes[t]].view(shapes[t]) for t in range(len(shapes))]
            for t in range(len(w)):
                w[t].copy_(torch.from_numpy(params0[t]).view(shapes[t]))
        else:
            w = [torch.from_numpy(p.copy()).to(DEV) for p in params0]
        comm.register_params(w)
        hg = torch.zeros(L, dtype=torch.float32).pin_memory()
        hw = torch.full((L,), float("nan"), dtype=torch.float32).pin_memory()
        for s in range(3):
            g = synth.grads(shapes, workers=1, step=s)
            for t in range(len(g[0])):
                hg[off[t]: off[t] + sizes[t]].copy_(torch.from_numpy(g[0][t]))
            orc.step(g, w_o, v_o, 0.1, 0.9, dtype)
            comm.step_host_packed(hg, hw, dtype, 0.1, 0.9)
            torch.cuda.synchronize()
            hwn = hw.numpy()
            for t in range(len(w_o)):
                assert_bitwise(hwn[off[t]: off[t] + sizes[t]].copy(), w_o[t], f"host w[{t}] step {s}")
    finally:
        comm.finalize()


def test_step_host_packed_pageable_params(cmn, orc):
    """Pageable host_params (synchronous D2H copies): same bits."""
    shapes = synth.resnet50_shapes()[:20]
    sizes = [synth.numel(s) for s in shapes]
    off, L = orc.layout(sizes)
    params0 = synth.params(shapes)
    w_o = [p.copy() for p in params0]
    v_o = [np.zeros_like(p) for p in params0]
    g = synth.grads(shapes, workers=1)
    orc.step(g, w_o, v_o, 0.1, 0.9, "fp32")
    comm = cmn.Comm.init(0, 1, 0)
    try:
        comm.register_params([torch.from_numpy(p.copy()).to(DEV) for p in params0])
        hg = torch.zeros(L, dtype=torch.float32).pin_memory()
        for t in range(len(sizes)):
            hg[off[t]: off[t] + sizes[t]].copy_(torch.from_numpy(g[0][t]))
        hw = torch.full((L,), float("nan"), dtype=torch.float32)      # pageable
        comm.step_host_packed(hg, hw, "fp32", 0.1, 0.9)
        torch.cuda.synchronize()
        for t in range(len(sizes)):
            assert_bitwise(hw.numpy()[off[t]: off[t] + sizes[t]].copy(), w_o[t], f"host w[{t}]")
    finally:
        comm.finalize()


@pytest.mark.parametrize("N,sched,flat,dtype", [(4, "pipelined", False, "fp32"), (3, "pipelined", True, "fp16"),
                                               (2, "serial", True, "fp32"), (8, "fused", False, "fp16"),
                                               (4, "pipelined7", True, "fp32")])
def test_step_host_packed_simulated(cmn, orc, N, sched, flat, dtype):
    """cmn_step_host_packed at N > 1 (simulated ranks), 3 steps: with the
    pipelined schedule the H2D of each piece feeds its pack and the D2H of
    its parameters follows its update on two copy streams; other schedules
    copy everything around the step.  Bit-exact with the oracle."""
    shapes = synth.resnet50_shapes()[:24] + RAGGED
    sizes = [synth.numel(s) for s in shapes]
    off, L = orc.layout(sizes)
    params0 = synth.params(shapes)
    w_o = [p.copy() for p in params0]
    v_o = [np.zeros_like(p) for p in params0]
    comm = cmn.Comm.simulated_world(N)
    try:
        if flat:
            buf = torch.zeros(off[len(sizes) - 1] + sizes[-1], dtype=torch.float32, device=DEV)
            w = [buf[off[t]: off[t] + sizes[t]].view(shapes[t]) for t in range(len(shapes))]
            for t in range(len(w)):
                w[t].copy_(torch.from_numpy(params0[t]).view(shapes[t]))
        else:
            w = to_dev(params0)
        comm.register_params(w)
        comm.set_fused_update(sched == "fused")
        comm.set_pipeline(0 if sched in ("serial", "fused") else int(sched[9:] or 4))
        hg = torch.zeros(N * L, dtype=torch.float32).pin_memory()
        hw = torch.full((L,), float("nan"), dtype=torch.float32).pin_memory()
        for step in range(3):
            g = synth.grads(shapes, workers=N, step=step)
            for i in range(N):
                for t in range(len(sizes)):
                    hg[i * L + off[t]: i * L + off[t] + sizes[t]].copy_(torch.from_numpy(g[i][t]))
            orc.step(g, w_o, v_o, 0.1, 0.9, dtype)
            comm.step_host_packed(hg, hw, dtype, 0.1, 0.9)
            torch.cuda.synchronize()
            for t in range(len(sizes)):
                assert_bitwise(hw.numpy()[off[t]: off[t] + sizes[t]].copy(), w_o[t], f"w[{t}] step {step}")
    finally:
        comm.finalize()


@pytest.mark.parametrize("dtype", ["fp32", "fp16"])
def test_nccl_comparison_plumbing_single_rank(cmn, orc, dtype):
    """CMN_ALGO_NCCL through a real (single-rank) NCCL communicator: dlopen of
    libnccl, ncclCommInitRank via the bootstrap path, ncclAllReduce on the
    packed buffer; a one-rank sum is exact, so the step is bit-exact.  (NCCL
    refuses two ranks on one GPU; its multi-rank numbers need >= 2 GPUs.)"""
    shapes = synth.mlp_shapes()
    g = synth.grads(shapes, workers=1)
    params0 = synth.params(shapes)
    ora, _, _ = run_oracle(orc, shapes, 1, dtype, [g], params0, 0.1, 0.9)
    comm = cmn.Comm.init(0, 1, 0)
    try:
        w = to_dev(params0)
        comm.register_params(w)
        comm.set_algo("nccl")
        comm.allreduce_grads(to_dev(g[0]), dtype)
        comm.update_momentum_sgd(0.1, 0.9)
        torch.cuda.synchronize()
        for t in range(len(w)):
            assert_bitwise(w[t].cpu().numpy().reshape(-1), ora[0]["w"][t], f"w[{t}]")
    finally:
        comm.finalize()


MANY = [(i % 7 + 1, 3) if i % 3 else (i % 5,) for i in range(600)]   # 600 tensors, incl. empty ones
TINY = [(1,), (2,), (3,)]                                               # L = 192: most chunks empty at N = 8


@pytest.mark.parametrize("shapes_name", ["many", "tiny"])
@pytest.mark.parametrize("N", [1, 3, 8])
def test_edge_layouts_all_schedules(cmn, orc, shapes_name, N):
    """600 tensors (3 launch groups of <= 256 grad pointers, zero-size tensors)
    and a 3-tensor model whose two-shot chunks are mostly empty at N = 8:
    unpipelined one-/two-shot, pipelined and sharded steps all bit-exact."""
    shapes = MANY if shapes_name == "many" else TINY
    grads = [synth.grads(shapes, workers=N, step=s, seed=11) for s in range(2)]
    params0 = synth.params(shapes, seed=11)
    for dtype in ("fp32", "fp16"):
        ora, _, _ = run_oracle(orc, shapes, N, dtype, grads, params0, 0.1, 0.9)
        for sched in ("oneshot", "twoshot", "pipelined", "sharded", "fused", "push"):
            comm = cmn.Comm.simulated_world(N) if N > 1 else cmn.Comm.init(0, 1, 0)
            try:
                w = to_dev(params0)
                comm.register_params(w)
                for s, g in enumerate(grads):
                    gd = [to_dev(gw) for gw in g] if N > 1 else to_dev(g[0])
                    if sched in ("oneshot", "twoshot"):
                        if N > 1:
                            comm.set_algo(sched)
                        comm.allreduce_grads(gd, dtype)
                        comm.update_momentum_sgd(0.1, 0.9)
                    elif sched == "pipelined":
                        comm.set_pipeline(3)
                        comm.step(gd, dtype, 0.1, 0.9)
                    elif sched in ("fused", "push"):
                        comm.set_fused_update("pull" if sched == "fused" else "push")
                        comm.step(gd, dtype, 0.1, 0.9)
                    else:
                        comm.step_sharded(gd, dtype, 0.1, 0.9)
                    torch.cuda.synchronize()
                    for t in range(len(w)):
                        assert_bitwise(w[t].cpu().numpy().reshape(-1), ora[s]["w"][t],
                                       f"{sched} {dtype} w[{t}] step {s}")
            finally:
                comm.finalize()


@pytest.mark.parametrize("dtype", ["fp32", "fp16"])
def test_nvls_single_rank(cmn, orc, dtype):
    """NEXT-3 plumbing on the one GPU gpurun provides (NVSwitch-attached):
    multicast object + bound allocation + unicast/multicast mappings, and
    the multimem.ld_reduce / multimem.st kernel.  With one rank the switch
    reduces a single copy, so the step must equal the oracle; checked
    bitwise except for signed zeros (an in-switch add may return +0 for -0),
    and within the tolerance gate."""
    shapes = synth.mlp_shapes() + RAGGED
    grads = [synth.grads(shapes, workers=1, step=s) for s in range(2)]
    params0 = synth.params(shapes)
    ora, off, L = run_oracle(orc, shapes, 1, dtype, grads, params0, 0.1, 0.9)
    comm = cmn.Comm.init(0, 1, 0)
    try:
        w = to_dev(params0)
        comm.register_params(w)
        try:
            comm.set_algo("nvls")
        except cmn.CmnError as e:
            if e.status_name == "CMN_ERR_UNSUPPORTED":
                pytest.skip(str(e))
            raise
        tdt = torch.float32 if dtype == "fp32" else torch.int16
        for s, g in enumerate(grads):
            comm.allreduce_grads(to_dev(g[0]), dtype)
            red = torch.empty(L, dtype=tdt, device=DEV)
            comm.copy_reduced(0, red)
            comm.update_momentum_sgd(0.1, 0.9)
            torch.cuda.synchronize()
            r = red.cpu().numpy()
            want = ora[s]["reduced"]
            if dtype == "fp32":
                r_bits, w_bits = r.view(np.uint32) & 0x7FFFFFFF, want.view(np.uint32) & 0x7FFFFFFF
                zero = (r_bits == 0) & (w_bits == 0)
            else:
                r_bits, w_bits = r.view(np.uint16) & 0x7FFF, want.view(np.uint16) & 0x7FFF
                zero = (r_bits == 0) & (w_bits == 0)
            assert np.array_equal(r.view(want.dtype)[~zero], want[~zero]), f"reduced step {s}"
            for t in range(len(w)):
                got = w[t].cpu().numpy().reshape(-1)
                assert np.allclose(got, ora[s]["w"][t], rtol=0, atol=0) or \
                    np.array_equal(got.view(np.uint32), ora[s]["w"][t].view(np.uint32)), f"w[{t}]"
    finally:
        comm.finalize()


def test_errors_are_loud(cmn):
    shapes = synth.mlp_shapes()
    comm = cmn.Comm.simulated_world(2)
    try:
        w = to_dev(synth.params(shapes))
        comm.register_params(w)
        with pytest.raises(cmn.CmnError) as e:
            comm.update_momentum_sgd(0.1, 0.9)
        assert e.value.status_name == "CMN_ERR_STATE"
        g = [to_dev(gw) for gw in synth.grads(shapes, workers=2)]
        bad = [list(gw) for gw in g]
        bad[1][0] = bad[1][0].view(-1)[1:]            # 4-byte offset: misaligned
        with pytest.raises(cmn.CmnError) as e:
            comm.allreduce_grads(bad, "fp32")
        assert e.value.status_name == "CMN_ERR_INVALID_ARG"
        with pytest.raises(cmn.CmnError):
            comm.allreduce_grads(g, 3)
        comm.allreduce_grads(g, "fp32")
        comm.update_momentum_sgd(0.1, 0.9)
        with pytest.raises(cmn.CmnError):
            comm.update_momentum_sgd(0.1, 0.9)         # consumed
        with pytest.raises(cmn.CmnError):
            comm.set_algo("nccl")                      # simulated: unsupported
        for bad_ctas in ((-1, 0), (0, 1025), (2000, 0)):
            with pytest.raises(cmn.CmnError) as e:
                comm.set_ctas(*bad_ctas)
            assert e.value.status_name == "CMN_ERR_INVALID_ARG"
    finally:
        comm.finalize()


def test_fp16_conversion_exhaustive_on_gpu(cmn, orc):
    """The GPU path's fp32->fp16 cast (inside k_pack) over a dense sweep of
    fp32 bit patterns vs the oracle's hand-written RNE (itself pinned to
    the compiler over all 2^32 inputs)."""
    single_rank_only(cmn)
    step = 4099  # coprime stride covering every exponent and many mantissas
    bits = (np.arange(0, 2 ** 32, step, dtype=np.uint64)).astype(np.uint32)
    x = bits.view(np.float32)
    n = x.size - (x.size % 4)
    x = x[:n]
    comm = cmn.Comm.init(0, 1, 0)
    try:
        w = [torch.zeros(n, dtype=torch.float32, device=DEV)]
        comm.register_params(w)
        comm.allreduce_grads([torch.from_numpy(x.copy()).to(DEV)], "fp16")
        p = torch.empty(n + (-n) % 64, dtype=torch.int16, device=DEV)
        comm.copy_packed(0, p)
        torch.cuda.synchronize()
        got = p.cpu().numpy().view(np.uint16)[:n]
        assert_bitwise(got, orc.f32_to_f16(x), "fp16 cast")
    finally:
        comm.finalize()


def test_launch_count(cmn):
    single_rank_only(cmn)
    shapes = synth.resnet50_shapes()
    comm = cmn.Comm.init(0, 1, 0)
    try:
        w = to_dev(synth.params(shapes))
        comm.register_params(w)
        g = to_dev(synth.grads(shapes, workers=1)[0])
        before = comm.kernel_launches
        comm.step(g, "fp32", 0.1, 0.9)
        assert comm.kernel_launches - before == 1      # one fused kernel at N = 1
    finally:
        comm.finalize()


def test_kernel_timing(cmn):
    """cmn_set_kernel_timing brackets each dominant-kernel launch: one per
    N = 1 step, one per piece of the pipelined schedule (internal stream),
    two per fused step; nothing while capturing a graph; results unchanged."""
    shapes = synth.resnet50_shapes()[:40]
    comm = cmn.Comm.init(0, 1, 0)
    try:
        comm.register_params(to_dev(synth.params(shapes)))
        g = to_dev(synth.grads(shapes, workers=1)[0])
        comm.set_kernel_timing(True)
        for _ in range(3):
            comm.step(g, "fp32", 0.1, 0.9)
        ms, n = comm.kernel_timing()
        assert n == 3 and ms > 0
        s2 = torch.cuda.Stream()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s2):
            comm.step(g, "fp32", 0.1, 0.9)
        graph.replay()
        torch.cuda.synchronize()
        assert comm.kernel_timing() == (0.0, 0)
        comm.set_kernel_timing(False)
        comm.step(g, "fp32", 0.1, 0.9)
        assert comm.kernel_timing() == (0.0, 0)
    finally:
        comm.finalize()
    comm = cmn.Comm.simulated_world(4)
    try:
        comm.register_params(to_dev(synth.params(shapes)))
        gs = [to_dev(gw) for gw in synth.grads(shapes, workers=4)]
        comm.set_pipeline(3)
        comm.set_kernel_timing(True)
        comm.step(gs, "fp16", 0.1, 0.9)
        assert comm.kernel_timing()[1] == 3
        comm.set_fused_update(True)
        comm.step(gs, "fp16", 0.1, 0.9)
        assert comm.kernel_timing()[1] == 2
    finally:
        comm.finalize()


@pytest.mark.parametrize("algo", ["oneshot", "twoshot"])
def test_fp16_rounded_once_on_gpu(cmn, algo):
    """The oracle pin test_fp16_payload_rounded_once on the CUDA path: the
    fp16 sum is accumulated in fp32 and rounded once (1 + 2^-11 + 2^-11 ->
    0x3c01; 65504 + 16 + 16 -> +inf), in both all-reduce kernels."""
    for vals, want in (([1.0, 2.0 ** -11, 2.0 ** -11], 0x3C01), ([65504.0, 16.0, 16.0], 0x7C00)):
        comm = cmn.Comm.simulated_world(3)
        try:
            comm.register_params([torch.zeros(1, device=DEV)])
            comm.set_algo(algo)
            comm.allreduce_grads([[torch.tensor([v], dtype=torch.float32, device=DEV)] for v in vals],
                                 "fp16")
            _, L = comm.layout()
            for r in range(3):
                q = torch.empty(L, dtype=torch.int16, device=DEV)
                comm.copy_reduced(r, q)
                assert int(q.cpu().numpy().view(np.uint16)[0]) == want, (vals, r)
        finally:
            comm.finalize()


@pytest.mark.parametrize("value_set", ["identical", "integer", "edge"])
@pytest.mark.parametrize("dtype", ["fp32", "fp16"])
def test_value_sets_every_schedule(cmn, orc, value_set, dtype):
    """The special value sets (identical workers, exact integer/dyadic set,
    planted inf / NaN / fp16-overflow / subnormal / tie values) through every
    N > 1 step schedule -- pipelined, fused pull, fused push, sharded --
    3 steps, bit-exact with the oracle (NaNs by position)."""
    shapes = synth.mlp_shapes()
    N = 4
    lr, mu = (2.0 ** -4, 2.0 ** -1) if value_set == "integer" else (0.1, 0.9)
    grads = [synth.grads(shapes, workers=N, step=s, value_set=value_set) for s in range(3)]
    params0 = synth.params(shapes, value_set="integer" if value_set == "integer" else "random")
    ora, _, _ = run_oracle(orc, shapes, N, dtype, grads, params0, lr, mu)
    for sched in ("pipelined", "pull", "push", "sharded"):
        comm = cmn.Comm.simulated_world(N)
        try:
            w = to_dev(params0)
            comm.register_params(w)
            comm.set_pipeline(3 if sched == "pipelined" else 0)
            comm.set_fused_update(sched if sched in ("pull", "push") else 0)
            for s, g in enumerate(grads):
                gd = [to_dev(gw) for gw in g]
                if sched == "sharded":
                    comm.step_sharded(gd, dtype, lr, mu)
                else:
                    comm.step(gd, dtype, lr, mu)
                torch.cuda.synchronize()
                for t in range(len(w)):
                    assert_bitwise(w[t].cpu().numpy().reshape(-1), ora[s]["w"][t],
                                   f"{sched} {value_set} {dtype} w[{t}] step {s}")
                    assert_bitwise(comm.momentum(t).cpu().numpy().reshape(-1), ora[s]["v"][t],
                                   f"{sched} {value_set} {dtype} v[{t}] step {s}")
        finally:
            comm.finalize()


@pytest.mark.parametrize("N,dtype,pieces", [(1, "fp32", 0), (1, "fp16", 0), (2, "fp32", 3),
                                            (4, "fp16", 4), (8, "fp32", 0), (3, "fp16", 2)])
def test_step_adam_parity(cmn, orc, N, dtype, pieces):
    """cmn_step_adam (NEXT-1 as a whole step): at N = 1 one kernel straight
    from the gradients, at N > 1 the pipelined schedule (or all-reduce then
    update with pieces = 0); w, m, v bit-exact with the oracle over 3 steps."""
    shapes = synth.resnet50_shapes()[:20] + RAGGED
    sizes = [synth.numel(s) for s in shapes]
    off, L = orc.layout(sizes)
    params0 = synth.params(shapes)
    w_o = [p.copy() for p in params0]
    m_o = [np.zeros_like(p) for p in params0]
    v_o = [np.zeros_like(p) for p in params0]
    comm = cmn.Comm.init(0, 1, 0) if N == 1 else cmn.Comm.simulated_world(N)
    try:
        w = to_dev(params0)
        comm.register_params(w)
        comm.set_pipeline(pieces)
        for step in range(1, 4):
            g = synth.grads(shapes, workers=N, step=step)
            red = orc.reduce_tree([orc.pack(gw, off, L, dtype) for gw in g], dtype)
            orc.update_adam(red, dtype, N, 1e-3, 0.9, 0.999, 1e-8, step, off, w_o, m_o, v_o)
            gd = to_dev(g[0]) if N == 1 else [to_dev(gw) for gw in g]
            comm.step_adam(gd, dtype, 1e-3, 0.9, 0.999, 1e-8, step)
            torch.cuda.synchronize()
            for t in range(len(w)):
                m, v = comm.adam_state(t)
                assert_bitwise(w[t].cpu().numpy().reshape(-1), w_o[t], f"adam w[{t}] step {step}")
                assert_bitwise(m.cpu().numpy().reshape(-1), m_o[t], f"adam m[{t}] step {step}")
                assert_bitwise(v.cpu().numpy().reshape(-1), v_o[t], f"adam v[{t}] step {step}")
    finally:
        comm.finalize()


@pytest.mark.parametrize("N", [1, 3])
def test_degenerate_models(cmn, orc, N):
    """Degenerate registrations: every tensor empty (L = 0: the step is a
    no-op that must not fail), and a single 1-element tensor (smaller than
    one vector, one chunk owner, pads everywhere) -- every schedule."""
    for shapes in ([(0,), (0, 5)], [(1,)]):
        grads = [synth.grads(shapes, workers=N, step=s) for s in range(2)]
        params0 = synth.params(shapes)
        ora, _, _ = run_oracle(orc, shapes, N, "fp32", grads, params0, 0.1, 0.9)
        for sched in (("serial", "pipelined", "pull", "push", "sharded") if N > 1 else ("direct",)):
            comm = cmn.Comm.init(0, 1, 0) if N == 1 else cmn.Comm.simulated_world(N)
            try:
                w = [torch.from_numpy(p.copy()).to(DEV).reshape(s) for p, s in zip(params0, shapes)]
                comm.register_params(w)
                comm.set_pipeline(2 if sched == "pipelined" else 0)
                comm.set_fused_update(sched if sched in ("pull", "push") else 0)
                for s, g in enumerate(grads):
                    gd = to_dev(g[0]) if N == 1 else [to_dev(gw) for gw in g]
                    if sched == "sharded":
                        comm.step_sharded(gd, "fp32", 0.1, 0.9)
                    else:
                        comm.step(gd, "fp32", 0.1, 0.9)
                    torch.cuda.synchronize()
                    for t in range(len(w)):
                        assert_bitwise(w[t].cpu().numpy().reshape(-1), ora[s]["w"][t], f"{shapes} {sched} w[{t}]")
            finally:
                comm.finalize()


@pytest.mark.parametrize("N,dtype,max_ctas", [(1, "fp32", 1), (1, "fp16", 5), (3, "fp32", 148),
                                              (3, "fp16", 7), (2, "fp32", 100000)])
def test_stream_ctas_parity(cmn, orc, N, dtype, max_ctas):
    """cmn_set_stream_ctas caps the pack / update / Adam grids; the capped
    CTAs stride over the work items.  Results are the oracle's, bitwise, for
    the whole-model call pair, the bucketed calls, and the Adam update (3
    steps each, ragged shapes spanning several items and tails)."""
    shapes = synth.resnet50_shapes()[:20] + RAGGED
    sizes = [synth.numel(s) for s in shapes]
    params0 = synth.params(shapes)
    grads = [synth.grads(shapes, workers=N, step=s) for s in range(3)]
    ora, off, L = run_oracle(orc, shapes, N, dtype, grads, params0, 0.1, 0.9)
    for bucketed in (False, True):
        comm = cmn.Comm.simulated_world(N) if N > 1 else cmn.Comm.init(0, 1, 0)
        try:
            w = to_dev(params0)
            comm.register_params(w)
            comm.set_stream_ctas(max_ctas)
            nb = comm.plan_buckets(1 << 18) if bucketed else 0
            for s, g in enumerate(grads):
                gd = [to_dev(gw) for gw in g] if N > 1 else to_dev(g[0])
                if bucketed:
                    table = comm.prepare(gd)
                    for b in range(nb):
                        comm.allreduce_bucket(b, table, dtype)
                    for b in range(nb):
                        comm.update_bucket(b, 0.1, 0.9)
                else:
                    comm.allreduce_grads(gd, dtype)
                    comm.update_momentum_sgd(0.1, 0.9)
                torch.cuda.synchronize()
                for t in range(len(w)):
                    what = f"{'bucketed' if bucketed else 'whole'} step {s}"
                    assert_bitwise(w[t].cpu().numpy().reshape(-1), ora[s]["w"][t], f"{what} w[{t}]")
                    assert_bitwise(comm.momentum(t).cpu().numpy().reshape(-1), ora[s]["v"][t],
                                   f"{what} v[{t}]")
        finally:
            comm.finalize()
    # Adam from the reduced buffer under the cap
    w_o = [p.copy() for p in params0]
    m_o = [np.zeros_like(p) for p in params0]
    v_o = [np.zeros_like(p) for p in params0]
    comm = cmn.Comm.simulated_world(N) if N > 1 else cmn.Comm.init(0, 1, 0)
    try:
        w = to_dev(params0)
        comm.register_params(w)
        comm.set_stream_ctas(max_ctas)
        for step, g in enumerate(grads, start=1):
            red = orc.reduce_tree([orc.pack(gw, off, L, dtype) for gw in g], dtype)
            orc.update_adam(red, dtype, N, 1e-3, 0.9, 0.999, 1e-8, step, off, w_o, m_o, v_o)
            comm.allreduce_grads([to_dev(gw) for gw in g] if N > 1 else to_dev(g[0]), dtype)
            comm.update_adam(1e-3, 0.9, 0.999, 1e-8, step)
            torch.cuda.synchronize()
            for t in range(len(w)):
                m, v = comm.adam_state(t)
                assert_bitwise(w[t].cpu().numpy().reshape(-1), w_o[t], f"adam w[{t}] step {step}")
                assert_bitwise(m.cpu().numpy().reshape(-1), m_o[t], f"adam m[{t}] step {step}")
                assert_bitwise(v.cpu().numpy().reshape(-1), v_o[t], f"adam v[{t}] step {step}")
    finally:
        comm.finalize()


def test_stream_ctas_invalid(cmn):
    comm = cmn.Comm.simulated_world(2)
    try:
        with pytest.raises(cmn.CmnError):
            comm.set_stream_ctas(-1)
        comm.set_stream_ctas(0)
    finally:
        comm.finalize()


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
@pytest.mark.parametrize("dtype", ["fp32", "fp16"])
def test_robustness_seeds_parity(cmn, orc, seed, dtype):
    """seeds 1-4 beside the base seed, MLP (config 1) and a
    ResNet-50 prefix with ragged tails, N = 2 and 5, both algorithms."""
    for shapes in (synth.mlp_shapes(), synth.resnet50_shapes()[:12] + [(4097,), (3,)]):
        for N in (2, 5):
            grads = [synth.grads(shapes, workers=N, step=s, seed=seed) for s in range(2)]
            params0 = synth.params(shapes, seed=seed)
            ora, _, _ = run_oracle(orc, shapes, N, dtype, grads, params0, 0.1, 0.9)
            for algo in ("oneshot", "twoshot"):
                gpu, _, _ = run_gpu(cmn, shapes, N, dtype, algo, grads, params0, 0.1, 0.9)
                compare(gpu, ora, N)


@pytest.mark.parametrize("per_tensor", ["0", "1"])
def test_step_host_packed_param_staging(cmn, orc, monkeypatch, per_tensor):
    """N = 1 e2e with separate parameter tensors: the updated params leave
    through the packed staging buffer (one D2H copy per piece; default) or
    per tensor (CMN_E2E_PER_TENSOR_D2H=1) -- same bits.  Re-registering a
    larger model re-sizes the staging buffer."""
    monkeypatch.setenv("CMN_E2E_PER_TENSOR_D2H", per_tensor)
    comm = cmn.Comm.init(0, 1, 0)
    try:
        for shapes in (synth.resnet50_shapes()[:9], RAGGED + synth.resnet50_shapes()[:40]):
            sizes = [synth.numel(s) for s in shapes]
            off, L = orc.layout(sizes)
            params0 = synth.params(shapes, seed=3)
            w_o = [p.copy() for p in params0]
            v_o = [np.zeros_like(p) for p in params0]
            comm.register_params([torch.from_numpy(p.copy()).to(DEV) for p in params0])
            hg = torch.zeros(L, dtype=torch.float32).pin_memory()
            hw = torch.full((L,), float("nan"), dtype=torch.float32).pin_memory()
            for s in range(2):
                g = synth.grads(shapes, workers=1, step=s, seed=3)
                for t in range(len(sizes)):
                    hg[off[t]: off[t] + sizes[t]].copy_(torch.from_numpy(g[0][t].reshape(-1)))
                orc.step(g, w_o, v_o, 0.1, 0.9, "fp32")
                comm.step_host_packed(hg, hw, "fp32", 0.1, 0.9)
                torch.cuda.synchronize()
                for t in range(len(sizes)):
                    assert_bitwise(hw.numpy()[off[t]: off[t] + sizes[t]].copy(), w_o[t], f"host w[{t}] step {s}")
    finally:
        comm.finalize()


@pytest.mark.parametrize("N,dtype", [(3, "fp32"), (5, "fp16"), (6, "fp32"), (7, "fp32")])
def test_average_by_division_every_kernel(cmn, orc, N, dtype):
    """Reading R3 ("dividing the sum by the number of
    replicas") at N that are not powers of two -- where r * fl(1/N) and r / N
    differ -- through every kernel that averages: cmn_unpack_avg_grads (the
    averaged gradient itself, vs the oracle's `avg` output), the update from
    the reduced buffer (serial and pipelined), the fused all-gather + update
    (pull and push), the sharded update and Adam, each bitwise vs the
    oracle."""
    shapes = RAGGED + [(1000,)]
    grads = synth.grads(shapes, workers=N, seed=11)
    params0 = synth.params(shapes, seed=11)
    w_o = [p.copy() for p in params0]
    v_o = [np.zeros_like(p) for p in params0]
    res = orc.step(grads, w_o, v_o, 0.1, 0.9, dtype, want_avg=True)
    # the oracle's average differs from the reciprocal product somewhere (the
    # case this test exists for)
    r = orc.f16_to_f32(res["reduced"]) if dtype == "fp16" else res["reduced"]
    recip = (r * np.float32(1.0 / N)).astype(np.float32)
    avg_flat = np.concatenate(res["avg"])
    off = res["off"]
    recip_flat = np.concatenate([recip[off[t]: off[t] + p.size] for t, p in enumerate(params0)])
    assert np.count_nonzero(avg_flat.view(np.uint32) != recip_flat.view(np.uint32)) > 0
    for mode in ("unpack", "serial", "pipelined", "fused", "push", "sharded"):
        comm = cmn.Comm.simulated_world(N)
        try:
            w = to_dev(params0)
            comm.register_params(w)
            gd = comm.prepare([to_dev(gw) for gw in grads])
            if mode == "unpack":
                comm.allreduce_grads(gd, dtype)
                out = [torch.empty_like(x) for x in w]
                comm.unpack_avg_grads(out)
                torch.cuda.synchronize()
                for t in range(len(w)):
                    assert_bitwise(out[t].cpu().numpy().reshape(-1), res["avg"][t], f"avg[{t}]")
                continue
            if mode == "serial":
                comm.allreduce_grads(gd, dtype)
                comm.update_momentum_sgd(0.1, 0.9)
            elif mode == "pipelined":
                comm.set_pipeline(3)
                comm.step(gd, dtype, 0.1, 0.9)
            elif mode in ("fused", "push"):
                comm.set_fused_update(1 if mode == "fused" else 2)
                comm.step(gd, dtype, 0.1, 0.9)
            else:
                comm.step_sharded(gd, dtype, 0.1, 0.9)
            torch.cuda.synchronize()
            for t in range(len(w)):
                assert_bitwise(w[t].cpu().numpy().reshape(-1), w_o[t], f"{mode} w[{t}]")
        finally:
            comm.finalize()
    # Adam from the reduced buffer
    sizes = [synth.numel(s) for s in shapes]
    w_a = [p.copy() for p in params0]
    m_a = [np.zeros_like(p) for p in params0]
    v_a = [np.zeros_like(p) for p in params0]
    orc.update_adam(res["reduced"], dtype, N, 1e-3, 0.9, 0.999, 1e-8, 1, orc.layout(sizes)[0], w_a, m_a, v_a)
    comm = cmn.Comm.simulated_world(N)
    try:
        w = to_dev(params0)
        comm.register_params(w)
        comm.allreduce_grads([to_dev(gw) for gw in grads], dtype)
        comm.update_adam(1e-3, 0.9, 0.999, 1e-8, 1)
        torch.cuda.synchronize()
        for t in range(len(w)):
            assert_bitwise(w[t].cpu().numpy().reshape(-1), w_a[t], f"adam w[{t}]")
    finally:
        comm.finalize()


@pytest.mark.parametrize("dtype", ["fp32", "fp16"])
def test_pack_16b_aligned_gradients_fallback(cmn, orc, dtype):
    """The pack's 256-bit path needs 32-byte aligned gradient pointers; the
    C ABI only requires 16 bytes.  Gradients placed at 16-byte (not 32-byte)
    offsets inside one allocation take the 128-bit path for those items:
    packed buffers, reduced buffers and w, v still bit-exact (N = 3)."""
    shapes = RAGGED + [(8192,), (64, 65)]
    N = 3
    grads = [synth.grads(shapes, workers=N, step=s, seed=13) for s in range(2)]
    params0 = synth.params(shapes, seed=13)
    ora, _, _ = run_oracle(orc, shapes, N, dtype, grads, params0, 0.1, 0.9)
    comm = cmn.Comm.simulated_world(N)
    try:
        w = to_dev(params0)
        comm.register_params(w)
        off, L = comm.layout()
        tdt = torch.float32 if dtype == "fp32" else torch.int16
        for s, g in enumerate(grads):
            gd = []
            for gw in g:
                views = []
                for t, x in enumerate(gw):
                    # every tensor 16 B past a 32-B boundary of its own buffer
                    buf = torch.empty(x.size + 8, dtype=torch.float32, device=DEV)
                    assert buf.data_ptr() % 32 == 0
                    v = buf[4: 4 + x.size]
                    assert v.data_ptr() % 32 == 16
                    v.copy_(torch.from_numpy(x.reshape(-1)))
                    views.append(v)
                gd.append(views)
            comm.allreduce_grads(gd, dtype)
            for r in range(N):
                p = torch.empty(L, dtype=tdt, device=DEV)
                comm.copy_packed(r, p)
                got = p.cpu().numpy()
                got = got.view(np.uint16) if dtype == "fp16" else got
                assert_bitwise(got, ora[s]["packed"][r], f"step {s} packed rank {r}")
            comm.update_momentum_sgd(0.1, 0.9)
            torch.cuda.synchronize()
            for t in range(len(w)):
                assert_bitwise(w[t].cpu().numpy().reshape(-1), ora[s]["w"][t], f"step {s} w[{t}]")
    finally:
        comm.finalize()


@pytest.mark.parametrize("N", [1, 3])
def test_checkpoint_resume_bitwise(cmn, orc, N):
    """SURVEY §5 checkpoint / resume: 2 steps, snapshot w and the library-
    owned momentum (cmn_get_momentum, read/write) to the host, finalize;
    a fresh communicator registers the restored w, writes the momentum back
    and takes 2 more steps -- bitwise equal to 4 uninterrupted oracle steps.
    The same for Adam's m and v (cmn_get_adam_state) with the step count
    continued by the caller."""
    shapes = synth.mlp_shapes() + [(4097,)]
    grads = [synth.grads(shapes, workers=N, step=s, seed=17) for s in range(4)]
    params0 = synth.params(shapes, seed=17)
    w_o = [p.copy() for p in params0]
    v_o = [np.zeros_like(p) for p in params0]
    for g in grads:
        orc.step(g, w_o, v_o, 0.1, 0.9, "fp32")

    def new_comm():
        return cmn.Comm.simulated_world(N) if N > 1 else cmn.Comm.init(0, 1, 0)

    def feed(g):
        return [to_dev(gw) for gw in g] if N > 1 else to_dev(g[0])

    comm = new_comm()
    try:
        w = to_dev(params0)
        comm.register_params(w)
        for g in grads[:2]:
            comm.step(feed(g), "fp32", 0.1, 0.9)
        torch.cuda.synchronize()
        ck_w = [x.cpu().clone() for x in w]
        ck_v = [comm.momentum(t).cpu().clone() for t in range(len(w))]
    finally:
        comm.finalize()
    comm = new_comm()
    try:
        w = [x.to(DEV) for x in ck_w]
        comm.register_params(w)                       # momentum starts at zero ...
        for t in range(len(w)):
            comm.momentum(t).copy_(ck_v[t].to(DEV))   # ... and is restored
        for g in grads[2:]:
            comm.step(feed(g), "fp32", 0.1, 0.9)
        torch.cuda.synchronize()
        for t in range(len(w)):
            assert_bitwise(w[t].cpu().numpy().reshape(-1), w_o[t].reshape(-1), f"resumed w[{t}]")
            assert_bitwise(comm.momentum(t).cpu().numpy().reshape(-1), v_o[t].reshape(-1), f"resumed v[{t}]")
    finally:
        comm.finalize()
    # Adam: m, v restored through cmn_get_adam_state, step count continued
    sizes = [synth.numel(s) for s in shapes]
    off = orc.layout(sizes)[0]
    wa = [p.copy() for p in params0]
    ma = [np.zeros_like(p) for p in params0]
    va = [np.zeros_like(p) for p in params0]
    for k, g in enumerate(grads):
        red = orc.reduce_tree([orc.pack(gw, off, orc.layout(sizes)[1], "fp32") for gw in g], "fp32")
        orc.update_adam(red, "fp32", N, 1e-3, 0.9, 0.999, 1e-8, k + 1, off, wa, ma, va)
    comm = new_comm()
    try:
        w = to_dev(params0)
        comm.register_params(w)
        for k, g in enumerate(grads[:2]):
            comm.step_adam(feed(g), "fp32", 1e-3, 0.9, 0.999, 1e-8, k + 1)
        torch.cuda.synchronize()
        ck_w = [x.cpu().clone() for x in w]
        ck = [tuple(s.cpu().clone() for s in comm.adam_state(t)) for t in range(len(w))]
    finally:
        comm.finalize()
    comm = new_comm()
    try:
        w = [x.to(DEV) for x in ck_w]
        comm.register_params(w)
        comm.step_adam(feed([[np.zeros_like(p) for p in params0] for _ in range(N)]), "fp32",
                       0.0, 0.9, 0.999, 1e-8, 1)        # allocates the state (alpha = 0: w unchanged)
        for t in range(len(w)):
            m_t, v_t = comm.adam_state(t)
            m_t.copy_(ck[t][0].to(DEV))
            v_t.copy_(ck[t][1].to(DEV))
        for t in range(len(w)):
            assert_bitwise(w[t].cpu().numpy().reshape(-1), ck_w[t].numpy().reshape(-1), "alpha=0 step")
        for k, g in enumerate(grads[2:]):
            comm.step_adam(feed(g), "fp32", 1e-3, 0.9, 0.999, 1e-8, k + 3)
        torch.cuda.synchronize()
        for t in range(len(w)):
            assert_bitwise(w[t].cpu().numpy().reshape(-1), wa[t].reshape(-1), f"resumed adam w[{t}]")
    finally:
        comm.finalize()


@pytest.mark.parametrize("sched", ["oneshot", "twoshot", "pipelined3", "fused", "push", "sharded",
                                   "buckets", "adam"])
@pytest.mark.parametrize("dtype", ["fp32", "fp16"])
@pytest.mark.parametrize("N", [3, 8])
def test_poisoned_buffers_every_schedule(cmn, orc, sched, dtype, N):
    """SURVEY §5's poisoned receive buffers: before every step the library's
    packed and reduced buffers of every rank (inbox slack included) are
    filled with 0x7FC07FC0 -- NaN as fp32 and as each fp16 half -- so a
    kernel that reads a location no kernel of the step wrote (a pad, a
    chunk tail, an inbox slot, the other parity) puts NaN into w.  Every
    schedule stays bit-exact with the oracle over 2 steps; in the emulated
    pass the barriers are live."""
    shapes = synth.mlp_shapes() + RAGGED
    sizes = [synth.numel(s) for s in shapes]
    off, L = orc.layout(sizes)
    params0 = synth.params(shapes)
    w_o = [p.copy() for p in params0]
    m_o = [np.zeros_like(p) for p in params0]
    v_o = [np.zeros_like(p) for p in params0]
    comm = cmn.Comm.simulated_world(N)
    try:
        w = to_dev(params0)
        comm.register_params(w)
        comm.set_algo("oneshot" if sched == "oneshot" else "twoshot")
        comm.set_pipeline(3 if sched == "pipelined3" else 0)
        comm.set_fused_update({"fused": 1, "push": 2}.get(sched, 0))
        nb = comm.plan_buckets(1 << 16) if sched == "buckets" else 0
        for step in range(1, 3):
            g = synth.grads(shapes, workers=N, step=step)
            red = orc.reduce_tree([orc.pack(gw, off, L, dtype) for gw in g], dtype)
            if sched == "adam":
                orc.update_adam(red, dtype, N, 1e-3, 0.9, 0.999, 1e-8, step, off, w_o, m_o, v_o)
            else:
                orc.update_momentum_sgd(red, dtype, N, 0.1, 0.9, off, w_o, v_o)
            gd = [to_dev(gw) for gw in g]
            comm.debug_fill_buffers()
            if sched == "adam":
                comm.step_adam(gd, dtype, 1e-3, 0.9, 0.999, 1e-8, step)
            elif sched == "sharded":
                comm.step_sharded(gd, dtype, 0.1, 0.9)
            elif sched == "buckets":
                for b in range(nb):
                    comm.allreduce_bucket(b, gd, dtype)
                for b in range(nb):
                    comm.update_bucket(b, 0.1, 0.9)
            else:
                comm.step(gd, dtype, 0.1, 0.9)
            torch.cuda.synchronize()
            comm.poll_error()
            for t in range(len(w)):
                assert_bitwise(w[t].cpu().numpy().reshape(-1), w_o[t], f"{sched} w[{t}] step {step}")
                if sched == "adam":
                    m, v = comm.adam_state(t)
                    assert_bitwise(v.cpu().numpy().reshape(-1), v_o[t], f"adam v[{t}] step {step}")
                else:
                    assert_bitwise(comm.momentum(t).cpu().numpy().reshape(-1), v_o[t],
                                   f"{sched} v[{t}] step {step}")
    finally:
        comm.finalize()


@pytest.mark.parametrize("dtype", ["fp32", "fp16"])
def test_poison_hook_reaches_the_buffers(cmn, dtype):
    """The poison test above is not vacuous: after a fill, every rank's
    packed and reduced buffers (what the kernels read) hold the NaN pattern
    in every element, and an update issued after the fill is refused."""
    shapes, N = synth.mlp_shapes(), 3
    comm = cmn.Comm.simulated_world(N)
    try:
        comm.register_params(to_dev(synth.params(shapes)))
        comm.allreduce_grads([to_dev(gw) for gw in synth.grads(shapes, workers=N)], dtype)
        comm.debug_fill_buffers()
        L = comm.layout()[1]
        tdt, pat = (torch.int32, 0x7FC07FC0) if dtype == "fp32" else (torch.int16, 0x7FC0)
        for r in range(N):
            for copy in (comm.copy_packed, comm.copy_reduced):
                q = torch.zeros(L, dtype=tdt, device=DEV)
                copy(r, q)
                assert bool((q == pat).all()), f"rank {r}: {copy.__name__} not poisoned"
        with pytest.raises(cmn.CmnError) as e:
            comm.update_momentum_sgd(0.1, 0.9)
        assert e.value.status_name == "CMN_ERR_STATE"
    finally:
        comm.finalize()


@pytest.mark.parametrize("dtype", ["fp32", "fp16"])
@pytest.mark.parametrize("sched", ["direct", "adam_direct", "oneshot", "twoshot", "pipelined3", "fused",
                                   "push", "sharded", "buckets", "adam"])
def test_guard_bands_untouched(cmn, orc, sched, dtype):
    """Out-of-bounds writes (the other half of what compute-sanitizer's
    memcheck would catch): every parameter tensor is a view into one
    allocation with 64-element guard bands of a canary pattern before,
    between and after the tensors (ragged sizes, so item tails end mid-band
    alignment).  The gradients sit between NaN canary bands the same way.
    After 2 steps of the schedule (N = 1 direct kernels, else N = 3) every
    canary word is intact, the gradients are unchanged (read-only) and w is
    bit-exact with the oracle (an out-of-bounds gradient read that reached
    the result would have made it NaN)."""
    shapes = synth.mlp_shapes() + RAGGED
    sizes = [synth.numel(s) for s in shapes]
    N = 1 if sched in ("direct", "adam_direct") else 3
    off, L = orc.layout(sizes)
    G = 64
    starts, pos = [], G
    for n in sizes:
        starts.append(pos)
        pos += -(-n // 8) * 8 + G          # 32-byte aligned starts, >= 64 canary words between
    canary = np.uint32(0x7FBADBAD)
    flat = torch.from_numpy(np.full(pos, canary, dtype=np.uint32).view(np.float32)).to(DEV)
    params0 = synth.params(shapes)
    w = []
    for t, n in enumerate(sizes):
        v = flat[starts[t]: starts[t] + n]
        v.copy_(torch.from_numpy(params0[t]))
        w.append(v.view(shapes[t]))
    mask = np.ones(pos, dtype=bool)
    for t, n in enumerate(sizes):
        mask[starts[t]: starts[t] + n] = False
    w_o = [p.copy() for p in params0]
    m_o = [np.zeros_like(p) for p in params0]
    v_o = [np.zeros_like(p) for p in params0]
    comm = cmn.Comm.init(0, 1, 0) if N == 1 else cmn.Comm.simulated_world(N)
    try:
        comm.register_params(w)
        if N > 1:
            comm.set_algo("oneshot" if sched == "oneshot" else "twoshot")
            comm.set_pipeline(3 if sched == "pipelined3" else 0)
            comm.set_fused_update({"fused": 1, "push": 2}.get(sched, 0))
        nb = comm.plan_buckets(1 << 16) if sched == "buckets" else 0
        adam = sched in ("adam", "adam_direct")
        for step in range(1, 3):
            g = synth.grads(shapes, workers=N, step=step)
            red = orc.reduce_tree([orc.pack(gw, off, L, dtype) for gw in g], dtype)
            if adam:
                orc.update_adam(red, dtype, N, 1e-3, 0.9, 0.999, 1e-8, step, off, w_o, m_o, v_o)
            else:
                orc.update_momentum_sgd(red, dtype, N, 0.1, 0.9, off, w_o, v_o)
            # gradients, too, live between NaN canary bands: an out-of-bounds
            # read that reached the result would turn it into NaN
            gflat = []
            gd = []
            for gw in g:
                fb = torch.from_numpy(np.full(pos, canary, dtype=np.uint32).view(np.float32)).to(DEV)
                views = []
                for t, n in enumerate(sizes):
                    fb[starts[t]: starts[t] + n].copy_(torch.from_numpy(gw[t]))
                    views.append(fb[starts[t]: starts[t] + n].view(shapes[t]))
                gflat.append((fb, fb.clone()))
                gd.append(views)
            gd = gd[0] if N == 1 else gd
            if adam:
                comm.step_adam(gd, dtype, 1e-3, 0.9, 0.999, 1e-8, step)
            elif sched == "sharded":
                comm.step_sharded(gd, dtype, 0.1, 0.9)
            elif sched == "buckets":
                for b in range(nb):
                    comm.allreduce_bucket(b, gd, dtype)
                for b in range(nb):
                    comm.update_bucket(b, 0.1, 0.9)
            else:
                comm.step(gd, dtype, 0.1, 0.9)
            torch.cuda.synchronize()
            for fb, before in gflat:          # the gradients are read-only (include/cmn.h)
                assert torch.equal(fb.view(torch.int32), before.view(torch.int32)), f"{sched}: grads written"
        comm.poll_error()
        bits = flat.cpu().numpy().view(np.uint32)
        bad = np.flatnonzero(bits[mask] != canary)
        assert bad.size == 0, f"{sched}: {bad.size} guard words overwritten"
        for t in range(len(w)):
            assert_bitwise(w[t].cpu().numpy().reshape(-1), w_o[t], f"{sched} w[{t}]")
    finally:
        comm.finalize()
