"""ctypes/numpy wrapper over the plain-C CPU oracle (oracle/cmn_oracle.c).

TEST INFRASTRUCTURE ONLY: importable from tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs.  The product package
(paper_1908_00213_b200) never imports this module, and this module never
imports the product package.

Each function names the step of SURVEY.md §8(c) c.1 (restated in
cmn_oracle.c's header and DESIGN.md §3) it implements.  All pins live in
tests/test_oracle_*.py; every function below is pinned (none is
"parity unpinned"); `update_adam` by the SPEC.md:463 example, its step-1
closed form and the constant-gradient multi-step closed form.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

FP32, FP16 = 0, 1
DTYPES = {"fp32": FP32, "fp16": FP16}
ALIGN = 64  # elements; reading c.2 #9

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_P = C.c_void_p
_I64P = C.POINTER(C.c_int64)


def build() -> str:
    """Compile liboracle.so (plain gcc; no CUDA)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return os.path.join(_HERE, "liboracle.so")


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        src = os.path.join(_HERE, "cmn_oracle.c")
        if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
            build()
        L = C.CDLL(path)
        L.orc_f32_to_f16.restype = C.c_uint16
        L.orc_f32_to_f16.argtypes = [C.c_float]
        L.orc_f16_to_f32.restype = C.c_float
        L.orc_f16_to_f32.argtypes = [C.c_uint16]
        L.orc_layout.restype = C.c_int64
        L.orc_layout.argtypes = [C.c_int, _I64P, C.c_int64, _I64P]
        L.orc_pack.restype = None
        L.orc_pack.argtypes = [C.c_int, _I64P, _I64P, C.c_int64, C.POINTER(_P), C.c_int, _P]
        L.orc_unpack_f32.restype = None
        L.orc_unpack_f32.argtypes = [C.c_int, _I64P, _I64P, _P, C.POINTER(_P)]
        L.orc_tree_sum.restype = C.c_float
        L.orc_tree_sum.argtypes = [C.POINTER(C.c_float), C.c_int, C.c_int]
        L.orc_reduce_tree.restype = C.c_int
        L.orc_reduce_tree.argtypes = [C.c_int, C.c_int64, C.POINTER(_P), C.c_int, _P]
        L.orc_update_momentum_sgd.restype = None
        L.orc_update_momentum_sgd.argtypes = [C.c_int, _I64P, _I64P, _P, C.c_int, C.c_int,
                                              C.c_float, C.c_float, C.POINTER(_P),
                                              C.POINTER(_P), C.POINTER(_P)]
        L.orc_update_adam.restype = None
        L.orc_update_adam.argtypes = [C.c_int, _I64P, _I64P, _P, C.c_int, C.c_int,
                                      C.c_float, C.c_float, C.c_float, C.c_float, C.c_int,
                                      C.POINTER(_P), C.POINTER(_P), C.POINTER(_P)]
        L.orc_exact_avg.restype = None
        L.orc_exact_avg.argtypes = [C.c_int, C.c_int64, C.POINTER(_P), _P, _P]
        L.orc_step.restype = C.c_int
        L.orc_step.argtypes = [C.c_int, C.c_int, _I64P, _I64P, C.c_int64, C.POINTER(_P),
                               C.c_int, C.c_float, C.c_float, C.POINTER(_P), C.POINTER(_P),
                               C.POINTER(_P), _P]
        L.orc_f32_to_f16_array.restype = None
        L.orc_f32_to_f16_array.argtypes = [_P, _P, C.c_int64]
        L.orc_f16_to_f32_array.restype = None
        L.orc_f16_to_f32_array.argtypes = [_P, _P, C.c_int64]
        _LIB = L
    return _LIB


# ----------------------------------------------------------------- helpers

def _dt(dtype) -> int:
    return DTYPES[dtype] if isinstance(dtype, str) else int(dtype)


def _np_comm(dtype):
    return np.float32 if _dt(dtype) == FP32 else np.uint16


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_I64P) if a.dtype == np.int64 else C.c_void_p(a.ctypes.data)


def _ptrs(arrs):
    return (_P * max(len(arrs), 1))(*[a.ctypes.data for a in arrs])


def _f32c(a) -> np.ndarray:
    a = np.asarray(a)
    assert a.dtype == np.float32 and a.flags.c_contiguous, "oracle inputs must be contiguous float32"
    return a


# ------------------------------------------------------------------- API

def f32_to_f16(x) -> np.ndarray:
    """fp32 -> fp16 bits (uint16), hand-written IEEE RNE (c.1 step 2)."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    out = np.empty(x.shape, dtype=np.uint16)
    lib().orc_f32_to_f16_array(C.c_void_p(x.ctypes.data), C.c_void_p(out.ctypes.data), x.size)
    return out


def f16_to_f32(h) -> np.ndarray:
    h = np.ascontiguousarray(np.asarray(h, dtype=np.uint16))
    out = np.empty(h.shape, dtype=np.float32)
    lib().orc_f16_to_f32_array(C.c_void_p(h.ctypes.data), C.c_void_p(out.ctypes.data), h.size)
    return out


def layout(sizes, align: int = ALIGN):
    """c.1 step 1: (offsets[T+1] int64, L)."""
    n = _i64(sizes)
    off = np.zeros(len(n) + 1, dtype=np.int64)
    L = lib().orc_layout(len(n), _ptr(n), align, _ptr(off))
    if L < 0:
        raise ValueError("bad layout input")
    return off, int(L)


def pack(grads, off, L, dtype="fp32") -> np.ndarray:
    """c.1 step 2: one worker's packed buffer (float32, or uint16 fp16 bits)."""
    g = [_f32c(x).reshape(-1) for x in grads]
    n = _i64([x.size for x in g])
    off = _i64(off)
    b = np.empty(L, dtype=_np_comm(dtype))
    lib().orc_pack(len(g), _ptr(n), _ptr(off), L, _ptrs(g), _dt(dtype), _ptr(b))
    return b


def unpack_f32(b, sizes, off):
    b = _f32c(b)
    out = [np.empty(int(s), dtype=np.float32) for s in sizes]
    lib().orc_unpack_f32(len(out), _ptr(_i64(sizes)), _ptr(_i64(off)), _ptr(b), _ptrs(out))
    return out


def tree_sum(x) -> np.float32:
    """Pairwise tree sum in rank order (c.1 step 3) of a 1-D float32 vector."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    return np.float32(lib().orc_tree_sum(x.ctypes.data_as(C.POINTER(C.c_float)), 0, x.size - 1))


def reduce_tree(bufs, dtype="fp32") -> np.ndarray:
    """c.1 steps 3-4: the reduced buffer every worker holds (comm dtype)."""
    ct = _np_comm(dtype)
    bufs = [np.ascontiguousarray(b) for b in bufs]
    assert all(b.dtype == ct for b in bufs)
    L = bufs[0].size
    r = np.empty(L, dtype=ct)
    rc = lib().orc_reduce_tree(len(bufs), L, _ptrs(bufs), _dt(dtype), _ptr(r))
    if rc != 0:
        raise RuntimeError("orc_reduce_tree failed")
    return r


def update_momentum_sgd(r, dtype, N, lr, mu, off, w, v, want_avg=False):
    """c.1 steps 5-6, in place on the lists of float32 arrays w and v."""
    r = np.ascontiguousarray(r)
    sizes = [x.size for x in w]
    a = [np.empty(s, dtype=np.float32) for s in sizes] if want_avg else None
    lib().orc_update_momentum_sgd(len(w), _ptr(_i64(sizes)), _ptr(_i64(off)), _ptr(r), _dt(dtype),
                                  int(N), float(lr), float(mu), _ptrs(w), _ptrs(v),
                                  _ptrs(a) if a is not None else None)
    return a


def update_adam(r, dtype, N, alpha, beta1, beta2, eps, step, off, w, m, v):
    """NEXT-1 fused Adam (bias-corrected), in place on w, m, v."""
    r = np.ascontiguousarray(r)
    sizes = [x.size for x in w]
    lib().orc_update_adam(len(w), _ptr(_i64(sizes)), _ptr(_i64(off)), _ptr(r), _dt(dtype), int(N),
                          float(alpha), float(beta1), float(beta2), float(eps), int(step),
                          _ptrs(w), _ptrs(m), _ptrs(v))


def exact_avg(packed_f32_bufs):
    """c.1 step 7: fp64 exact average and condition magnitude m."""
    bufs = [_f32c(b) for b in packed_f32_bufs]
    L = bufs[0].size
    avg = np.empty(L, dtype=np.float64)
    mag = np.empty(L, dtype=np.float64)
    lib().orc_exact_avg(len(bufs), L, _ptrs(bufs), _ptr(avg), _ptr(mag))
    return avg, mag


def step(grads_per_worker, w, v, lr, mu, dtype="fp32", align: int = ALIGN, want_avg=False):
    """One full synchronous step (c.1 steps 1-6) for N simulated workers.

    grads_per_worker[i][t]: float32 arrays; w, v: lists of float32 arrays updated
    in place.  Returns dict(off, L, reduced, avg)."""
    N = len(grads_per_worker)
    T = len(w)
    sizes = [x.size for x in w]
    off, L = layout(sizes, align)
    flat = [_f32c(g).reshape(-1) for gw in grads_per_worker for g in gw]
    assert len(flat) == N * T
    r = np.empty(L, dtype=_np_comm(dtype))
    a = [np.empty(s, dtype=np.float32) for s in sizes] if want_avg else None
    rc = lib().orc_step(N, T, _ptr(_i64(sizes)), _ptr(off), L, _ptrs(flat), _dt(dtype),
                        float(lr), float(mu), _ptrs(w), _ptrs(v),
                        _ptrs(a) if a is not None else None, _ptr(r))
    if rc != 0:
        raise RuntimeError("orc_step failed")
    return {"off": off, "L": L, "reduced": r, "avg": a}


def step_threaded(grads_per_worker, w, v, lr, mu, dtype="fp32", threads: int = 0):
    """The same step with the elements partitioned across host threads
    ("elementwise partition across nproc threads,
    which gives bit-identical output").  Timing aid for bench.py only.

    Every quantity of c.1 steps 2-6 for element j depends only on element j
    of each worker's gradient and of w, v (pack/cast, tree sum over workers,
    1/N, momentum update), so the flattened parameter space is cut into
    `threads` contiguous element ranges (split inside tensors where needed)
    and each range is run through the unchanged single-threaded `step` on its
    own thread (ctypes releases the GIL during the C call).  w and v are
    updated in place; the reduced buffer and its layout are not returned
    (each range has its own).  Arithmetic is exactly `step`'s."""
    import concurrent.futures as cf
    threads = threads or os.cpu_count() or 1
    N = len(grads_per_worker)
    wf = [np.asarray(x).reshape(-1) for x in w]
    vf = [np.asarray(x).reshape(-1) for x in v]
    for x in wf + vf:  # reshape must be a view: w, v are updated in place
        _f32c(x)
    gf = [[_f32c(g).reshape(-1) for g in gw] for gw in grads_per_worker]
    total = sum(x.size for x in wf)
    per = -(-total // threads) if total else 0
    parts = []  # per thread: list of (tensor index, lo, hi)
    t, k = 0, 0
    for _ in range(threads):
        need, part = per, []
        while need > 0 and t < len(wf):
            take = min(need, wf[t].size - k)
            if take > 0:
                part.append((t, k, k + take))
            need -= take
            k += take
            if k >= wf[t].size:
                t, k = t + 1, 0
        if part:
            parts.append(part)

    def run(part):
        g = [[gf[i][t][lo:hi] for (t, lo, hi) in part] for i in range(N)]
        step(g, [wf[t][lo:hi] for (t, lo, hi) in part], [vf[t][lo:hi] for (t, lo, hi) in part],
             lr, mu, dtype)

    with cf.ThreadPoolExecutor(max_workers=max(1, len(parts))) as ex:
        list(ex.map(run, parts))
    return len(parts)
