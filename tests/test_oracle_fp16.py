"""Pins for the oracle's fp32 <-> fp16 conversion (c.1 step 2; reading R4:
IEEE binary16 round-to-nearest-even, no FTZ, overflow to inf), the paper's
"half-precision floats for communication" (App. A.1).

Pinned against two independent IEEE implementations: the compiler's
_Float16 / F16C conversion (all 2^32 inputs) and numpy's float16."""
import os
import shutil
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.filterwarnings("ignore:overflow encountered in cast")

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.slow
def test_f32_to_f16_exhaustive_vs_compiler(orc, tmp_path):
    """All 2^32 fp32 patterns vs gcc's _Float16 conversion (F16C), ~5 s."""
    odir = os.path.dirname(orc.build())
    exe = tmp_path / "f16x"
    src = os.path.join(HERE, "helpers", "f16_exhaustive.c")
    built = False
    for gcc in filter(None, {shutil.which("gcc"), shutil.which(os.environ.get("CC", "gcc"))}):
        for flags in (["-O2", "-fopenmp", "-mf16c"], ["-O2", "-mf16c"], ["-O2"]):
            rc = subprocess.run([gcc, *flags, "-o", str(exe), src, f"-L{odir}", "-loracle",
                                 f"-Wl,-rpath,{odir}"], capture_output=True).returncode
            if rc == 0:
                built = True
                break
        if built:
            break
    assert built, "could not compile the exhaustive fp16 checker"
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-2000:]
    assert "mismatches=0" in out.stdout


def test_f32_to_f16_vs_numpy_sample(orc):
    rng = np.random.default_rng(1)
    bits = rng.integers(0, 2**32, size=2_000_000, dtype=np.uint64).astype(np.uint32)
    x = bits.view(np.float32)
    mine = orc.f32_to_f16(x)
    ref = x.astype(np.float16).view(np.uint16)
    nan = np.isnan(x)
    assert np.array_equal(mine[~nan], ref[~nan])
    # NaN stays NaN with its sign (compared by class, reading R4)
    assert np.all((mine[nan] & 0x7C00) == 0x7C00) and np.all(mine[nan] & 0x3FF)
    assert np.array_equal(mine[nan] >> 15, ref[nan] >> 15)


def test_f16_special_values(orc):
    cases = {
        65504.0: 0x7BFF,          # max half
        65519.996: 0x7BFF,        # just below the overflow tie
        65520.0: 0x7C00,          # tie between 65504 and 65536 -> even -> inf
        -70000.0: 0xFC00,
        2.0 ** -14: 0x0400,       # min normal
        2.0 ** -24: 0x0001,       # min subnormal
        2.0 ** -25: 0x0000,       # tie with 0 -> even -> 0
        3 * 2.0 ** -26: 0x0001,   # 0.75 * 2^-24 -> 1 unit
        3 * 2.0 ** -25: 0x0002,   # 1.5 units -> tie -> even 2
        1.0 + 2.0 ** -11: 0x3C00, # tie -> even (1.0)
        1.0 + 3 * 2.0 ** -11: 0x3C02,
        -0.0: 0x8000,
    }
    x = np.array(list(cases.keys()), dtype=np.float32)
    got = orc.f32_to_f16(x)
    assert [int(v) for v in got] == list(cases.values())


def test_f16_to_f32_all_patterns(orc):
    h = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    mine = orc.f16_to_f32(h)
    ref = h.view(np.float16).astype(np.float32)
    nan = np.isnan(ref)
    assert np.array_equal(mine[~nan].view(np.uint32), ref[~nan].view(np.uint32))
    assert np.all(np.isnan(mine[nan]))
