"""Pins for the oracle's all-reduce (c.1 steps 3-4): the sum over workers
("obtain and distribute the sum of gradients", §6.1.2) in a
fixed pairwise-tree order (reading R2), fp16 payload rounded once (R4).

Pins: hand-derived tree-shape cases (tests/golden/tree_order.json), SPEC's
worked example, brute-force exact sums with the closed-form error bound,
identical-worker and integer-set invariants."""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _hexf(s):
    return np.array([int(s, 16)], dtype=np.uint32).view(np.float32)[0]


def test_tree_shape_golden(orc):
    cases = json.load(open(os.path.join(GOLD, "tree_order.json")))["cases"]
    for c in cases:
        x = np.array([_hexf(h) for h in c["inputs_hex"]], dtype=np.float32)
        got = orc.tree_sum(x)
        assert got.view(np.uint32) == int(c["tree"], 16), c["derivation"]
        # the same inputs distributed over workers through reduce_tree
        bufs = [np.array([v], dtype=np.float32) for v in x]
        r = orc.reduce_tree(bufs, "fp32")
        assert r.view(np.uint32)[0] == int(c["tree"], 16)


def test_spec_allreduce_example(orc):
    ex = json.load(open(os.path.join(GOLD, "spec_examples.json")))["allreduce"]
    bufs = [np.array(w, dtype=np.float32) for w in ex["workers"]]
    assert list(orc.reduce_tree(bufs, "fp32")) == ex["expected_sum"]


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 6, 7, 8])
def test_reduce_bruteforce_exact_bound(orc, N):
    """|tree - exact| <= ceil(log2 N) * 2^-24 * sum|x| (pairwise-sum bound,
    depth ceil(log2 N)), exact sum in rationals."""
    rng = np.random.default_rng(100 + N)
    L = 64
    bufs = [(rng.standard_normal(L) * 10.0 ** rng.integers(-3, 3, L)).astype(np.float32) for _ in range(N)]
    r = orc.reduce_tree(bufs, "fp32")
    depth = math.ceil(math.log2(N)) if N > 1 else 0
    for j in range(L):
        exact = sum(Fraction(float(b[j])) for b in bufs)
        absum = sum(abs(Fraction(float(b[j]))) for b in bufs)
        err = abs(Fraction(float(r[j])) - exact)
        assert err <= Fraction(depth, 2 ** 24) * absum * (1 + Fraction(1, 2 ** 20))


@pytest.mark.parametrize("N", [1, 2, 4, 8])
def test_identical_workers_return_gradient(orc, N):
    """N identical workers -> r / N == g bit-exact (north star invariant)."""
    shapes = synth.mlp_shapes()
    sizes = [synth.numel(s) for s in shapes]
    off, L = orc.layout(sizes)
    g = synth.grads(shapes, workers=N, value_set="identical")
    packed = [orc.pack(gw, off, L, "fp32") for gw in g]
    r = orc.reduce_tree(packed, "fp32")
    a = (r / np.float32(N)).astype(np.float32)
    assert np.array_equal(a.view(np.uint32), packed[0].view(np.uint32))
    # fp16 payload: tree(N * h) = N*h exactly, rounded once -> h; avg -> widen(h)
    p16 = [orc.pack(gw, off, L, "fp16") for gw in g]
    r16 = orc.reduce_tree(p16, "fp16")
    a16 = orc.f16_to_f32(r16) / np.float32(N)
    assert np.array_equal(a16.astype(np.float32), orc.f16_to_f32(p16[0]))


@pytest.mark.parametrize("dtype", ["fp32", "fp16"])
def test_integer_set_is_exact(orc, dtype):
    """Integer grads in [-128,127]: every partial sum (|s| <= 1024) is exact in
    both fp32 and fp16, so r equals the integer sum exactly."""
    shapes = synth.mlp_shapes()
    sizes = [synth.numel(s) for s in shapes]
    off, L = orc.layout(sizes)
    for N in (2, 3, 8):
        g = synth.grads(shapes, workers=N, value_set="integer")
        packed = [orc.pack(gw, off, L, dtype) for gw in g]
        r = orc.reduce_tree(packed, dtype)
        rf = r if dtype == "fp32" else orc.f16_to_f32(r)
        ints = sum(orc.pack(gw, off, L, "fp32").astype(np.int64) for gw in g)
        assert np.array_equal(rf.astype(np.int64), ints)


def test_fp16_tolerance_gate_vs_exact(orc):
    """fp16 path: |a - abar| <= 2e-3*m + 2^-24 (north-star tolerance,
    condition-aware reading R16)."""
    shapes = synth.mlp_shapes()
    sizes = [synth.numel(s) for s in shapes]
    off, L = orc.layout(sizes)
    for N in (2, 8):
        g = synth.grads(shapes, workers=N)
        p32 = [orc.pack(gw, off, L, "fp32") for gw in g]
        p16 = [orc.pack(gw, off, L, "fp16") for gw in g]
        a16 = orc.f16_to_f32(orc.reduce_tree(p16, "fp16")).astype(np.float64) / N
        a32 = orc.reduce_tree(p32, "fp32").astype(np.float64) / N
        avg, mag = orc.exact_avg(p32)
        assert np.all(np.abs(a16 - avg) <= 2e-3 * mag + 2.0 ** -24)
        assert np.all(np.abs(a32 - avg) <= 1e-5 * mag)


def test_exact_avg_closed_form(orc):
    x = [np.array([1.0, -2.0, 0.5], np.float32), np.array([3.0, 2.0, -0.25], np.float32)]
    avg, mag = orc.exact_avg(x)
    assert list(avg) == [2.0, 0.0, 0.125]
    assert list(mag) == [2.0, 2.0, 0.375]


def test_fp16_payload_rounded_once(orc):
    """Reading R4: fp16 payloads are accumulated in fp32 and the reduced sum
    is rounded to fp16 exactly once.  Hand-derived case where rounding per
    addition (an fp16 accumulator, or re-rounding per hop) gives another
    answer: 1 + 2^-11 + 2^-11 with fp16 ulp(1) = 2^-10.
      once:     fl16(1 + 2^-11 + 2^-11) = fl16(1 + 2^-10) = 0x3c01
      per add:  fl16(1 + 2^-11) = 1 (tie to even), then again 1 = 0x3c00
    Also 65504 + 16 + 16 (fp16 max, half an ulp = 16): once -> 65536 -> +inf
    (0x7c00); per add: 65504 + 16 ties to even 65504, then 65504 (0x7bff)."""
    cases = [([1.0, 2.0 ** -11, 2.0 ** -11], 0x3C01),
             ([65504.0, 16.0, 16.0], 0x7C00)]
    for vals, want in cases:
        bufs = [np.array([v], dtype=np.float32) for v in vals]
        packed = [orc.pack([b], np.array([0, 64]), 64, "fp16") for b in bufs]
        r = orc.reduce_tree(packed, "fp16")
        assert int(r.view(np.uint16)[0]) == want, (vals, hex(int(r.view(np.uint16)[0])))
