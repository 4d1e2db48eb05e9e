"""Host-side checks of the C ABI (no GPU needed): the library loads and
exports every symbol include/cmn.h declares, the binding declares them all,
the host-only plan helpers agree with the oracle's layout, and the compute
entry points fail loudly (CMN_ERR_CUDA) when no sm_100 device is present."""
import os
import re

import pytest
import torch

import synth
from paper_1908_00213_b200 import cmn

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cmn.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cmn_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1908_00213_b200 import build
    build.build()
    return cmn.lib()


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ("cmn_init", "cmn_register_params", "cmn_allreduce_grads", "cmn_update_momentum_sgd"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    for s in declared_symbols():
        assert hasattr(lib, s), f"{s} declared in cmn.h but not exported"


def test_binding_covers_every_declared_symbol():
    bound = {name for name, _, _ in cmn.SIGNATURES}
    assert set(declared_symbols()) == bound


def test_version(lib):
    assert lib.cmn_version() == 1


@pytest.mark.parametrize("workload", ["mlp", "r50"])
def test_plan_layout_matches_oracle(lib, orc, workload):
    shapes = synth.WORKLOADS[workload]()
    off, L, h = cmn.plan_layout(shapes)
    ooff, oL = orc.layout([synth.numel(s) for s in shapes])
    assert off == list(ooff) and L == oL
    # structure hash: same shapes -> same hash; transposed shape -> different
    _, _, h2 = cmn.plan_layout(shapes)
    assert h == h2
    sw = list(shapes)
    sw[0] = tuple(reversed(sw[0]))
    _, _, h3 = cmn.plan_layout(sw)
    assert h3 != h or sw[0] == shapes[0]


def test_plan_layout_rejects_bad_input(lib):
    with pytest.raises(cmn.CmnError) as e:
        cmn.plan_layout([])
    assert e.value.status == 1
    with pytest.raises(cmn.CmnError):
        cmn.plan_layout([(3, -1)])


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 8])
def test_plan_chunks_partition(lib, N):
    for L in (0, 64, 640, 89792, 25557056):
        s, e = cmn.plan_chunks(L, N)
        assert s[0] == 0 and e[-1] == L
        for r in range(N):
            assert s[r] <= e[r]
            assert s[r] % 64 == 0
            if r:
                assert s[r] == e[r - 1]
        c = e[0] - s[0]
        assert c == min(L, -(-(-(-L // N)) // 64) * 64)


def test_r50_chunks_match_survey(lib):
    # L/8 = 3,194,632 -> chunks of 3,194,688, last 3,194,240
    s, e = cmn.plan_chunks(25557056, 8)
    assert e[0] - s[0] == 3194688 and e[7] - s[7] == 3194240


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback(lib):
    with pytest.raises(cmn.CmnError) as e:
        cmn.Comm.simulated_world(2)
    assert e.value.status_name == "CMN_ERR_CUDA"
    with pytest.raises(cmn.CmnError):
        cmn.Comm.init(0, 1, 0)
    with pytest.raises(cmn.CmnError) as e:
        cmn.Comm.emulated_world(2)
    assert e.value.status_name == "CMN_ERR_CUDA"


def test_invalid_world(lib):
    import ctypes as C
    h = C.c_void_p()
    assert lib.cmn_init_simulated(9, 0, C.byref(h)) == 1
    assert lib.cmn_init_simulated(0, 0, C.byref(h)) == 1
    assert lib.cmn_init_emulated(9, 0, C.byref(h)) == 1
    assert lib.cmn_init_emulated(0, 0, C.byref(h)) == 1


@pytest.mark.parametrize("bucket_mb", [0, 1, 4, 8, 16, 25, 1000])
def test_bucket_plan(bucket_mb):
    """cmn_plan_bucket_ranges (host only) against a plain re-statement of its
    definition in include/cmn.h: contiguous reverse-order ranges covering
    every tensor once, each holding at most bucket_bytes of fp32 gradients
    unless it is a single larger tensor, and maximal (the next tensor would
    not fit); bucket_bytes == 0 gives one bucket."""
    import synth
    from paper_1908_00213_b200 import cmn
    sizes = [synth.numel(s) for s in synth.resnet50_shapes()]
    cap = bucket_mb << 20
    plan = cmn.plan_bucket_ranges(sizes, cap)
    assert plan[0][1] == len(sizes) and plan[-1][0] == 0
    for (b0, e0), (b1, e1) in zip(plan, plan[1:]):
        assert e1 == b0                              # contiguous, reverse order
    for b, e in plan:
        nbytes = 4 * sum(sizes[b:e])
        assert e > b
        if cap == 0:
            assert (b, e) == (0, len(sizes))
            continue
        assert nbytes <= cap or e - b == 1
        if b > 0:
            assert nbytes + 4 * sizes[b - 1] > cap    # maximal
    if cap == 0:
        assert len(plan) == 1


# ---- property-based host-logic checks (random shapes, sizes, world sizes)
from hypothesis import given, settings, strategies as st  # noqa: E402

_dims = st.lists(st.integers(min_value=0, max_value=70), min_size=1, max_size=3)


@settings(max_examples=200, deadline=None)
@given(shapes=st.lists(_dims, min_size=1, max_size=40))
def test_plan_layout_matches_oracle_random(lib, orc, shapes):
    """The library's layout (a0) equals the oracle's on random shapes, zero-size
    dimensions included; offsets are 64-aligned and non-decreasing."""
    shapes = [tuple(s) for s in shapes]
    sizes = [int(__import__("numpy").prod(s)) for s in shapes]
    off, L, _ = cmn.plan_layout(shapes)
    o_off, o_L = orc.layout(sizes)
    assert list(off) == [int(x) for x in o_off] and L == o_L
    assert all(o % 64 == 0 for o in off)
    assert all(off[t + 1] - off[t] >= sizes[t] for t in range(len(sizes)))


@settings(max_examples=300, deadline=None)
@given(blocks=st.integers(min_value=0, max_value=1 << 22), N=st.integers(min_value=1, max_value=8))
def test_plan_chunks_partition_random(lib, blocks, N):
    """§8(e): chunks partition [0, L) into N contiguous 64-aligned pieces of
    align64(ceil(L/N)) elements (the last one shorter, possibly empty)."""
    L = 64 * blocks
    s, e = cmn.plan_chunks(L, N)
    c = min(L, -(-(-(-L // N)) // 64) * 64)
    pos = 0
    for r in range(N):
        assert s[r] == pos and s[r] % 64 == 0
        assert e[r] - s[r] == max(0, min(c, L - pos))
        pos = e[r]
    assert pos == L


@settings(max_examples=200, deadline=None)
@given(sizes=st.lists(st.integers(min_value=0, max_value=3_000_000), min_size=1, max_size=60),
       cap=st.sampled_from([0, 1, 4096, 1 << 16, 1 << 20, 4 << 20, 25 << 20]))
def test_bucket_plan_random(sizes, cap):
    """a4 buckets on random tensor sizes: contiguous reverse-order ranges
    covering every tensor once, within the byte cap unless a single tensor,
    and maximal (the next tensor would not fit)."""
    plan = cmn.plan_bucket_ranges(sizes, cap)
    assert plan[0][1] == len(sizes) and plan[-1][0] == 0
    for (b0, _), (_, e1) in zip(plan, plan[1:]):
        assert e1 == b0
    for b, e in plan:
        assert e > b
        nbytes = 4 * sum(sizes[b:e])
        if cap == 0:
            assert (b, e) == (0, len(sizes))
            continue
        assert nbytes <= cap or e - b == 1
        if b > 0:
            assert nbytes + 4 * sizes[b - 1] > cap
