"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds ONLY input generation (a counter-based hash -> numbers)
and workload shape tables.  It contains none of the method's arithmetic
(no packing, no reduction, no update), so both sides of every parity check
may use it without sharing code with each other (task rule ③).

Generator (stated again in DESIGN.md §4):

    mix(x)  = splitmix64 finaliser of x + 0x9E3779B97F4A7C15
    key     = mix(mix(mix(mix(mix(seed) ^ set) ^ step) ^ worker) ^ tensor)
    h_k     = mix(key ^ k)                         (k = element index in tensor)
    u_k     = ((h_k >> 40) - 2^23) * 2^-23         in [-1, 1), exactly 24 bits
    e_t     = 4 + (mix(seed ^ t) mod 13)           in [4, 16]
    grad    = u_k * 2^-e_t                         (exact in fp32)
    param   = u_k * 2^-3   (set = SET_PARAM, worker = 0, step = 0)

Value sets: "random" (above), "identical" (every worker draws worker = 0),
"integer" (grad = signed top byte of h_k, in [-128, 127]; params in
2^-4 * [-128, 127]), "edge" (random, with inf / NaN / fp16-overflow /
fp16-subnormal / signed-zero values planted at fixed positions of tensor 0).
"""
from __future__ import annotations

import numpy as np

from .workloads import WORKLOADS, mlp_shapes, resnet50_shapes, numel  # noqa: F401

BASE_SEED = 190800213
SET_IDS = {"random": 1, "identical": 2, "integer": 3, "edge": 4}
SET_PARAM = 100

_M64 = (1 << 64) - 1
_GOLD = 0x9E3779B97F4A7C15
_C1 = 0xBF58476D1CE4E5B9
_C2 = 0x94D049BB133111EB


def mix(x: int) -> int:
    """splitmix64 on a Python int (scalar path)."""
    z = (x + _GOLD) & _M64
    z = ((z ^ (z >> 30)) * _C1) & _M64
    z = ((z ^ (z >> 27)) * _C2) & _M64
    return z ^ (z >> 31)


def _mix_np(x: np.ndarray) -> np.ndarray:
    z = x + np.uint64(_GOLD)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(_C1)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(_C2)
    return z ^ (z >> np.uint64(31))


def stream_key(seed: int, set_id: int, step: int, worker: int, tensor: int) -> int:
    k = mix(seed & _M64)
    for v in (set_id, step, worker, tensor):
        k = mix(k ^ (v & _M64))
    return k


def hashes(key: int, n: int) -> np.ndarray:
    k = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return _mix_np(k ^ np.uint64(key))


def unit24(h: np.ndarray) -> np.ndarray:
    """((h >> 40) - 2^23) * 2^-23 as float32 (exact)."""
    i = (h >> np.uint64(40)).astype(np.int64) - (1 << 23)
    return (i.astype(np.float32) * np.float32(2.0 ** -23)).astype(np.float32)


def tensor_exponent(seed: int, t: int) -> int:
    return 4 + (mix((seed ^ t) & _M64) % 13)


def grad_tensor(n: int, t: int, *, seed: int = BASE_SEED, step: int = 0,
                worker: int = 0, value_set: str = "random") -> np.ndarray:
    """Worker `worker`'s gradient of tensor t at `step` (float32, n elements)."""
    sid = SET_IDS[value_set]
    wk = 0 if value_set == "identical" else worker
    key = stream_key(seed, sid, step, wk, t)
    h = hashes(key, n)
    if value_set == "integer":
        return ((h >> np.uint64(56)).astype(np.int64) - 128).astype(np.float32)
    g = unit24(h) * np.float32(2.0 ** -tensor_exponent(seed, t))
    g = g.astype(np.float32)
    if value_set == "edge" and t == 0 and n > 0:
        plant = np.array([np.inf, -np.inf, np.nan, 65520.0, -70000.0, 65504.0,
                          2.0 ** -25, 3.0 * 2.0 ** -26, 2.0 ** -24, -2.0 ** -20,
                          0.0, -0.0, 1e-30, 2.0 ** -14, 2.0 ** -14 - 2.0 ** -25,
                          1.0 + 2.0 ** -11], dtype=np.float32)
        pos = (np.arange(len(plant)) * 37 + worker * 5) % n
        g[pos[: min(len(plant), n)]] = plant[: min(len(plant), n)]
    return g


def param_tensor(n: int, t: int, *, seed: int = BASE_SEED, value_set: str = "random") -> np.ndarray:
    key = stream_key(seed, SET_PARAM, 0, 0, t)
    h = hashes(key, n)
    if value_set == "integer":
        i = ((h >> np.uint64(56)).astype(np.int64) - 128).astype(np.float32)
        return (i * np.float32(2.0 ** -4)).astype(np.float32)
    return (unit24(h) * np.float32(2.0 ** -3)).astype(np.float32)


def grads(shapes, *, workers: int, seed: int = BASE_SEED, step: int = 0,
          value_set: str = "random"):
    """list over workers of list over tensors of float32 arrays."""
    sizes = [numel(s) for s in shapes]
    return [[grad_tensor(n, t, seed=seed, step=step, worker=i, value_set=value_set)
             for t, n in enumerate(sizes)] for i in range(workers)]


def params(shapes, *, seed: int = BASE_SEED, value_set: str = "random"):
    return [param_tensor(numel(s), t, seed=seed, value_set=value_set)
            for t, s in enumerate(shapes)]
