"""Exact-arithmetic helpers for pinning the oracle (independent of it).

round_f32(q) rounds a rational to the nearest binary32 (ties to even) by
comparing exact distances of neighbouring candidates -- no reliance on
fp64 intermediate rounding (which would double-round)."""
from fractions import Fraction

import numpy as np


def frac(x) -> Fraction:
    return Fraction(float(x))


def round_f32(q: Fraction) -> np.float32:
    c = np.float32(float(q))
    if not np.isfinite(c):
        return c
    cands = {c, np.nextafter(c, np.float32(np.inf)), np.nextafter(c, np.float32(-np.inf))}
    best = None
    for x in cands:
        if not np.isfinite(x):
            continue
        d = abs(frac(x) - q)
        if best is None or d < best[0]:
            best = (d, x)
        elif d == best[0]:
            # tie: even significand (last bit of the binary32 pattern clear)
            xb = int(np.array(x, np.float32).view(np.uint32))
            if xb & 1 == 0:
                best = (d, x)
    return np.float32(best[1])


def fma_f32(a, b, c) -> np.float32:
    """Correctly rounded a*b + c for binary32 inputs."""
    return round_f32(frac(a) * frac(b) + frac(c))


def add_f32(a, b) -> np.float32:
    return round_f32(frac(a) + frac(b))
