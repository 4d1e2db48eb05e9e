"""Pins for the oracle's average + momentum-SGD update (c.1 steps 5-6):
"calculates the average of gradients by dividing the sum by the number of
replicas, and updates its own replica" (§6.1.2), momentum
form v = mu v + g, w -= lr v (reading R6: explicit fma).

Pins: SPEC's worked examples, momentum=0 reduces to SGD, correctly-rounded
fma checked in exact rationals, the n=2 g/3g example, integer/dyadic
exactness over 3 steps, and the fp32 tolerance gate."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import synth
from helpers.exact import fma_f32, round_f32

SPEC = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _one_tensor_step(orc, g_list, w, v, lr, mu, dtype="fp32"):
    res = orc.step([[np.asarray(g, np.float32)] for g in g_list], [w], [v], lr, mu, dtype, want_avg=True)
    return res["avg"][0]


def test_spec_sgd_example(orc):
    ex = SPEC["sgd"]
    w = np.array([ex["w0"]], np.float32)
    v = np.zeros(1, np.float32)
    _one_tensor_step(orc, [[ex["g"]]], w, v, ex["lr"], ex["mu"])
    assert abs(float(w[0]) - ex["expected_w"][0]) < 1e-6


def test_spec_momentum_two_steps(orc):
    ex = SPEC["momentum"]
    w = np.array([ex["w0"]], np.float32)
    v = np.zeros(1, np.float32)
    for want in ex["expected_w"]:
        _one_tensor_step(orc, [[ex["g"]]], w, v, ex["lr"], ex["mu"])
        assert abs(float(w[0]) - want) < 2e-7 * 4


def test_spec_average_example(orc):
    ex = SPEC["average"]
    g = synth.grad_tensor(1000, 3)
    w = np.zeros(1000, np.float32)
    v = np.zeros(1000, np.float32)
    a = _one_tensor_step(orc, [g * np.float32(f) for f in ex["factor_workers"]], w, v, 0.1, 0.0)
    assert np.array_equal(a, (g * np.float32(ex["expected_factor"])).astype(np.float32))


def test_average_divides_by_replica_count_n3(orc):
    """Hand-derived pin of reading R3 at N = 3 ("dividing
    the sum by the number of replicas"), where dividing and multiplying by
    the rounded reciprocal differ.  Workers send 5, 0, 0: the tree sum is 5
    exactly.  5/3 = 1.0101010...(binary); rounded to 24 bits the discarded
    tail 0.1010... of an ulp is above a half -> 1.01010101010101010101011
    = 0x3FD55555 (1.66666662693...).  The reciprocal route gives
    5 * RN(1/3) = 5 * 0x3EAAAAAB = 55924055 / 2^25 = 1.66666671633...,
    which rounds to 0x3FD55556 -- so a dropped division shows up here."""
    w = np.zeros(1, np.float32)
    v = np.zeros(1, np.float32)
    a = _one_tensor_step(orc, [[5.0], [0.0], [0.0]], w, v, 0.0, 0.0)
    assert int(a.view(np.uint32)[0]) == 0x3FD55555
    assert int(v.view(np.uint32)[0]) == 0x3FD55555      # mu = 0: v' = a


def test_momentum_zero_is_sgd_exact_rounding(orc):
    """mu = 0: v' = a, w' = round(w - lr*a) correctly rounded (one fma)."""
    rng = np.random.default_rng(7)
    n = 300
    g = rng.standard_normal(n).astype(np.float32)
    w0 = rng.standard_normal(n).astype(np.float32)
    v0 = rng.standard_normal(n).astype(np.float32)   # ignored when mu = 0
    w, v = w0.copy(), v0.copy()
    lr = np.float32(0.0123)
    _one_tensor_step(orc, [g], w, v, lr, 0.0)
    assert np.array_equal(v, g)
    for k in range(n):
        assert w[k] == round_f32(Fraction(float(w0[k])) - Fraction(float(lr)) * Fraction(float(g[k])))


@pytest.mark.parametrize("N", [1, 2, 3, 5, 6, 7, 8])
def test_update_is_correctly_rounded_fma(orc, N):
    """v' = RN(mu v + a), w' = RN(w - lr v') checked in exact rationals, with
    a = RN(r / N) ("dividing the sum by the number of replicas",
    PAPER.md:453-454; reading R3) and r the oracle's reduced sum (pinned
    elsewhere)."""
    rng = np.random.default_rng(11 + N)
    n = 200
    gs = [rng.standard_normal(n).astype(np.float32) for _ in range(N)]
    w0 = rng.standard_normal(n).astype(np.float32)
    v0 = rng.standard_normal(n).astype(np.float32)
    lr, mu = np.float32(0.1), np.float32(0.9)
    w, v = w0.copy(), v0.copy()
    res = orc.step([[g] for g in gs], [w], [v], lr, mu, "fp32", want_avg=True)
    r = res["reduced"]
    for k in range(n):
        a = round_f32(Fraction(float(r[k])) / N)
        assert res["avg"][0][k] == a
        vn = fma_f32(mu, v0[k], a)
        wn = fma_f32(-lr, vn, w0[k])
        assert v[k] == vn and w[k] == wn


@pytest.mark.parametrize("dtype", ["fp32", "fp16"])
def test_integer_dyadic_three_steps_exact(orc, dtype):
    """Integer grads, w in 2^-4 Z, lr = 2^-4, mu = 2^-1, N in {2, 4}: all
    operations exact, so w, v equal the exact rational recurrence."""
    shapes = synth.mlp_shapes()
    for N in (2, 4):
        w = synth.params(shapes, value_set="integer")
        v = [np.zeros_like(x) for x in w]
        wq = [x.astype(np.float64) for x in w]
        vq = [np.zeros_like(x) for x in wq]
        for s in range(3):
            g = synth.grads(shapes, workers=N, step=s, value_set="integer")
            orc.step(g, w, v, 2.0 ** -4, 2.0 ** -1, dtype)
            for t in range(len(w)):
                mean = sum(g[i][t].astype(np.float64) for i in range(N)) / N
                vq[t] = 0.5 * vq[t] + mean
                wq[t] = wq[t] - vq[t] / 16
                assert np.array_equal(v[t].astype(np.float64), vq[t])
                assert np.array_equal(w[t].astype(np.float64), wq[t])


def test_fp32_tolerance_gate_r50_sample(orc):
    """Random set, N = 8, a slice of ResNet-50's tensors: |a - abar| <= 1e-5 m."""
    shapes = synth.resnet50_shapes()[:12]
    sizes = [synth.numel(s) for s in shapes]
    N = 8
    g = synth.grads(shapes, workers=N)
    w = synth.params(shapes)
    v = [np.zeros_like(x) for x in w]
    res = orc.step(g, w, v, 0.1, 0.9, "fp32", want_avg=True)
    off, L = res["off"], res["L"]
    p32 = [orc.pack(gw, off, L, "fp32") for gw in g]
    avg, mag = orc.exact_avg(p32)
    for t, n in enumerate(sizes):
        a = res["avg"][t].astype(np.float64)
        assert np.all(np.abs(a - avg[off[t]: off[t] + n]) <= 1e-5 * mag[off[t]: off[t] + n])


def test_replicas_bitwise_equal_and_deterministic(orc):
    shapes = synth.mlp_shapes()
    g = synth.grads(shapes, workers=4)
    outs = []
    for _ in range(2):
        w = synth.params(shapes)
        v = [np.zeros_like(x) for x in w]
        for s in range(2):
            orc.step(g, w, v, 0.1, 0.9, "fp16")
        outs.append(np.concatenate(w + v).view(np.uint32))
    assert np.array_equal(outs[0], outs[1])


def test_adam_spec_example_and_step1_closed_form(orc):
    ex = SPEC["adam"]
    off, L = orc.layout([1])
    w = [np.array([ex["w0"]], np.float32)]
    m = [np.zeros(1, np.float32)]
    v = [np.zeros(1, np.float32)]
    r = np.array([ex["g"]], np.float32)
    orc.update_adam(r, "fp32", 1, ex["alpha"], ex["beta1"], ex["beta2"], ex["eps"], 1, off, w, m, v)
    assert abs(float(w[0][0]) - ex["expected_w"]) < 1e-6
    # step-1 closed form: m = (1-b1) g, v = (1-b2) g^2, dw = alpha*g/(|g| + eps/sqrt(1-b2))
    rng = np.random.default_rng(5)
    g = (rng.standard_normal(500) * 1e-2).astype(np.float32)
    off, L = orc.layout([500])
    w = [np.ones(500, np.float32)]
    m = [np.zeros(500, np.float32)]
    v = [np.zeros(500, np.float32)]
    orc.update_adam(g, "fp32", 1, 1e-3, 0.9, 0.999, 1e-8, 1, off, w, m, v)
    g64 = g.astype(np.float64)
    c1 = 1.0 - float(np.float32(0.9))      # the fp32 hyper-parameters' exact values
    c2 = 1.0 - float(np.float32(0.999))
    assert np.allclose(m[0], c1 * g64, rtol=1e-6, atol=0)
    assert np.allclose(v[0], c2 * g64 * g64, rtol=1e-6, atol=0)
    dw = 1.0 - w[0].astype(np.float64)
    want = 1e-3 * g64 / (np.abs(g64) + 1e-8 / np.sqrt(c2))
    assert np.allclose(dw, want, rtol=2e-3, atol=1e-7)


@pytest.mark.parametrize("steps", [1, 3, 10])
def test_adam_constant_gradient_trajectory_closed_form(orc, steps):
    """Multi-step pin of the Adam oracle (bias correction, step index): with a
    constant gradient g, m_t = (1-b1^t) g and v_t = (1-b2^t) g^2 exactly in
    real arithmetic, so each step moves w by alpha*g / (|g| + eps/sqrt(1-b2^t)).
    The fp64 sum of those steps must match the fp32 oracle to ~1e-5 relative
    (a wrong power, an off-by-one step index or a missing correction fails)."""
    rng = np.random.default_rng(21)
    g = (rng.standard_normal(400) * 10.0 ** rng.integers(-4, 0, 400)).astype(np.float32)
    off, L = orc.layout([400])
    w = [np.zeros(400, np.float32)]
    m = [np.zeros(400, np.float32)]
    v = [np.zeros(400, np.float32)]
    a, b1, b2, eps = 1e-3, 0.9, 0.999, 1e-8
    for t in range(1, steps + 1):
        orc.update_adam(g, "fp32", 1, a, b1, b2, eps, t, off, w, m, v)
    g64 = g.astype(np.float64)
    b2f = float(np.float32(b2))
    want = -sum(a * g64 / (np.abs(g64) + eps / np.sqrt(1.0 - b2f ** t)) for t in range(1, steps + 1))
    assert np.allclose(w[0], want, rtol=2e-5 * steps, atol=1e-9)
    b1f = float(np.float32(b1))
    assert np.allclose(m[0], (1 - b1f ** steps) * g64, rtol=1e-5, atol=0)
    assert np.allclose(v[0], (1 - b2f ** steps) * g64 * g64, rtol=1e-4, atol=0)


@pytest.mark.parametrize("dtype", ["fp32", "fp16"])
@pytest.mark.parametrize("threads", [1, 3, 8, 17])
def test_threaded_partition_bitwise_equal(orc, dtype, threads):
    """the elementwise partition across host threads
    (bench.py's cpu_baseline timing aid) gives bit-identical w, v.  Ragged
    shapes force ranges that split tensors and threads > elements of some
    ranges; 3 steps carry momentum across the partition."""
    shapes = [(5,), (4097,), (3, 7), (1,), (64, 65), (0,), (12289,)]
    N = 3
    w1 = synth.params(shapes, seed=5)
    w2 = [x.copy() for x in w1]
    v1 = [np.zeros_like(x) for x in w1]
    v2 = [np.zeros_like(x) for x in w1]
    for s in range(3):
        g = synth.grads(shapes, workers=N, step=s, seed=5)
        orc.step(g, w1, v1, 0.1, 0.9, dtype)
        orc.step_threaded(g, w2, v2, 0.1, 0.9, dtype, threads=threads)
    for a, b in zip(w1 + v1, w2 + v2):
        assert a.tobytes() == b.tobytes()
