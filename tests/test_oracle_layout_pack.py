"""Pins for the oracle's layout and pack/unpack (c.1 steps 1-2).

Layout: reading R9 (align-64 offsets, zero pads) on the parameter order of a
model traversal (§3.2).  Pins: hand-worked MLP offsets
(tests/golden/layouts.json), ResNet-50 totals, closed-form properties, and a
brute-force index-mapping check that encodes (t, k) into every element."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.filterwarnings("ignore:overflow encountered in cast")

import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "layouts.json")))


def test_mlp_layout_golden(orc):
    g = GOLD["mlp"]
    sizes = [synth.numel(s) for s in synth.mlp_shapes()]
    assert sizes == g["sizes"] and sum(sizes) == g["P"]
    off, L = orc.layout(sizes)
    assert list(off) == g["offsets"] and L == g["L"]


def test_r50_layout_totals(orc):
    g = GOLD["r50"]
    sizes = [synth.numel(s) for s in synth.resnet50_shapes()]
    assert len(sizes) == g["T"] and sum(sizes) == g["P"]
    off, L = orc.layout(sizes)
    assert L == g["L"]


def test_layout_properties(orc):
    rng = np.random.default_rng(3)
    for align in (1, 4, 64, 128):
        sizes = list(rng.integers(0, 300, size=40)) + [0, 1, 63, 64, 65]
        off, L = orc.layout(sizes, align)
        assert off[0] == 0 and L == off[-1]
        for t, n in enumerate(sizes):
            assert off[t] % align == 0
            gap = off[t + 1] - off[t] - n
            assert 0 <= gap < align


def test_pack_index_mapping_bruteforce(orc):
    """Encode (t, k) as a float32-exact integer 1000*t + k + 1 and decode."""
    sizes = [5, 1, 64, 0, 130, 7]
    g = [np.array([1000 * t + k + 1 for k in range(n)], dtype=np.float32) for t, n in enumerate(sizes)]
    off, L = orc.layout(sizes)
    b = orc.pack(g, off, L, "fp32")
    owner = {}
    for t, n in enumerate(sizes):
        for k in range(n):
            owner[off[t] + k] = (t, k)
    for j in range(L):
        if j in owner:
            t, k = owner[j]
            assert b[j] == 1000 * t + k + 1
        else:
            assert b[j] == 0.0 and not np.signbit(b[j])   # pads are +0
    # inverse mapping
    back = orc.unpack_f32(b, sizes, off)
    for x, y in zip(g, back):
        assert np.array_equal(x, y)


def test_pack_fp16_is_elementwise_cast(orc):
    shapes = synth.mlp_shapes()
    g = synth.grads(shapes, workers=1, value_set="edge")[0]
    sizes = [synth.numel(s) for s in shapes]
    off, L = orc.layout(sizes)
    b16 = orc.pack(g, off, L, "fp16")
    b32 = orc.pack(g, off, L, "fp32")
    assert b16.dtype == np.uint16 and b16.size == L
    ref = b32.astype(np.float16).view(np.uint16)        # numpy's IEEE RNE cast
    nan = np.isnan(b32)
    assert np.array_equal(b16[~nan], ref[~nan])
    pad = np.ones(L, bool)
    for t, n in enumerate(sizes):
        pad[off[t]: off[t] + n] = False
    assert np.all(b16[pad] == 0)
