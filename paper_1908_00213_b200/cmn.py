"""Thin ctypes binding over libcmn.so (include/cmn.h), same names as the C ABI.

Argument marshalling only: every step of the path runs in the library's
sm_100a kernels.  PyTorch is used for device memory, streams and the
torch.distributed bootstrap group -- never for the method's arithmetic.
There is no fallback: if libcmn.so is missing or no sm_100 device is
present, every compute call raises CmnError.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Sequence

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcmn.so")

FP32, FP16 = 0, 1
ALGO_AUTO, ALGO_ONESHOT, ALGO_TWOSHOT, ALGO_NCCL, ALGO_NVLS = 0, 1, 2, 3, 4
_ALGOS = {"auto": 0, "oneshot": 1, "twoshot": 2, "nccl": 3, "nvls": 4}
_DTYPES = {"fp32": FP32, "fp16": FP16, "float32": FP32, "float16": FP16}
STATUS = {0: "CMN_OK", 1: "CMN_ERR_INVALID_ARG", 2: "CMN_ERR_CUDA", 3: "CMN_ERR_NCCL",
          4: "CMN_ERR_BOOTSTRAP", 5: "CMN_ERR_MISMATCH", 6: "CMN_ERR_TIMEOUT",
          7: "CMN_ERR_STATE", 8: "CMN_ERR_OOM", 9: "CMN_ERR_UNSUPPORTED"}

# (name, restype, argtypes) -- every symbol include/cmn.h declares.
_P = C.c_void_p
_PP = C.POINTER(C.c_void_p)
_I64P = C.POINTER(C.c_int64)
AllgatherFn = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)
SIGNATURES = [
    ("cmn_init", C.c_int, [C.c_int, C.c_int, C.c_int, AllgatherFn, _P, _PP]),
    ("cmn_init_simulated", C.c_int, [C.c_int, C.c_int, _PP]),
    ("cmn_init_emulated", C.c_int, [C.c_int, C.c_int, _PP]),
    ("cmn_debug_fill_buffers", C.c_int, [_P, C.c_uint32, _P]),
    ("cmn_finalize", C.c_int, [_P]),
    ("cmn_register_params", C.c_int, [_P, C.c_int, C.POINTER(C.c_int), _I64P, _PP]),
    ("cmn_get_layout", C.c_int, [_P, _I64P, _I64P]),
    ("cmn_allreduce_grads", C.c_int, [_P, _PP, C.c_int, _P]),
    ("cmn_update_momentum_sgd", C.c_int, [_P, C.c_float, C.c_float, _P]),
    ("cmn_step", C.c_int, [_P, _PP, C.c_int, C.c_float, C.c_float, _P]),
    ("cmn_step_sharded", C.c_int, [_P, _PP, C.c_int, C.c_float, C.c_float, _P]),
    ("cmn_step_host", C.c_int, [_P, _PP, _PP, C.c_int, C.c_float, C.c_float, _P]),
    ("cmn_step_host_packed", C.c_int, [_P, _P, _P, C.c_int, C.c_float, C.c_float, _P]),
    ("cmn_unpack_avg_grads", C.c_int, [_P, _PP, _P]),
    ("cmn_update_adam", C.c_int, [_P, C.c_float, C.c_float, C.c_float, C.c_float, C.c_int, _P]),
    ("cmn_step_adam", C.c_int, [_P, _PP, C.c_int, C.c_float, C.c_float, C.c_float, C.c_float, C.c_int,
                                _P]),
    ("cmn_plan_buckets", C.c_int, [_P, C.c_size_t, C.POINTER(C.c_int)]),
    ("cmn_get_bucket", C.c_int, [_P, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("cmn_allreduce_bucket", C.c_int, [_P, C.c_int, _PP, C.c_int, _P]),
    ("cmn_update_bucket", C.c_int, [_P, C.c_int, C.c_float, C.c_float, _P]),
    ("cmn_set_algo", C.c_int, [_P, C.c_int, C.c_size_t]),
    ("cmn_set_pipeline", C.c_int, [_P, C.c_int]),
    ("cmn_set_fused_update", C.c_int, [_P, C.c_int]),
    ("cmn_set_ctas", C.c_int, [_P, C.c_int, C.c_int]),
    ("cmn_set_stream_ctas", C.c_int, [_P, C.c_int]),
    ("cmn_set_kernel_timing", C.c_int, [_P, C.c_int]),
    ("cmn_get_kernel_timing", C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_int)]),
    ("cmn_set_timeout", C.c_int, [_P, C.c_uint32]),
    ("cmn_get_momentum", C.c_int, [_P, C.c_int, _PP]),
    ("cmn_get_adam_state", C.c_int, [_P, C.c_int, _PP, _PP]),
    ("cmn_copy_packed", C.c_int, [_P, C.c_int, _P, _P]),
    ("cmn_copy_reduced", C.c_int, [_P, C.c_int, _P, _P]),
    ("cmn_poll_error", C.c_int, [_P]),
    ("cmn_kernel_launches", C.c_uint64, [_P]),
    ("cmn_last_error", C.c_char_p, []),
    ("cmn_version", C.c_int, []),
    ("cmn_plan_layout", C.c_int, [C.c_int, C.POINTER(C.c_int), _I64P, _I64P, _I64P,
                                  C.POINTER(C.c_uint64)]),
    ("cmn_plan_chunks", C.c_int, [C.c_int64, C.c_int, _I64P, _I64P]),
    ("cmn_plan_bucket_ranges", C.c_int, [C.c_int, _I64P, C.c_size_t, C.POINTER(C.c_int),
                                         C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("cmn_bootstrap_verify", C.c_int, [C.c_int, C.c_int, AllgatherFn, _P, C.c_uint64]),
    ("cmn_share_fd", C.c_int, [C.c_int, C.c_int, AllgatherFn, _P, C.c_int, C.POINTER(C.c_int)]),
]

_LIB = None


class CmnError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        self.status = status
        self.status_name = STATUS.get(status, str(status))
        super().__init__(f"{where}: {self.status_name}: {msg}")


def lib() -> C.CDLL:
    """Load the in-tree libcmn.so (raises if it was not built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise CmnError(2, "load", f"{LIB_PATH} missing -- run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _LIB = L
    return _LIB


def _check(rc: int, where: str):
    if rc != 0:
        raise CmnError(rc, where, lib().cmn_last_error().decode(errors="replace"))


def _dt(dtype) -> int:
    return _DTYPES[dtype] if isinstance(dtype, str) else int(dtype)


def _ptr_array(ptrs: Sequence[int]):
    arr = (C.c_void_p * max(len(ptrs), 1))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr


def _shapes_args(shapes):
    nd = (C.c_int * len(shapes))(*[len(s) for s in shapes])
    flat = [int(d) for s in shapes for d in s]
    dims = (C.c_int64 * max(len(flat), 1))(*flat)
    return nd, dims


def _stream(stream) -> int:
    if stream is None:
        # torch's current stream of the current device, read without
        # building a torch.cuda.Stream object (~0.3 us instead of ~3 us)
        import torch
        return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _data_ptrs(tensors, device=None) -> list:
    """Raw pointers of fp32 tensors.  The kernels treat every pointer as
    contiguous fp32 on the communicator's device, so anything else is
    refused here (CMN_ERR_INVALID_ARG) instead of faulting on the GPU:
    device=int requires CUDA tensors on that device, device="cpu" host
    tensors (the host-buffer step), None skips the placement check."""
    out = []
    for t in tensors:
        if isinstance(t, int):
            out.append(t)
            continue
        if t.dtype != _torch().float32:
            raise CmnError(1, "marshal", f"tensors must be float32 (got {t.dtype})")
        if not t.is_contiguous():
            raise CmnError(1, "marshal", "tensors must be contiguous")
        if device == "cpu":
            if t.is_cuda:
                raise CmnError(1, "marshal", "host-buffer calls take CPU (pinned) tensors")
        elif device is not None:
            if not t.is_cuda or t.device.index != device:
                raise CmnError(1, "marshal", f"tensors must be on cuda:{device} (got {t.device})")
        out.append(t.data_ptr())
    return out


def _torch():
    import torch
    return torch


class PtrTable:
    """Pre-marshalled pointer table (gradients registered once and reused
    every step, as a framework's persistent .grad buffers are): building it
    costs ~1 us per tensor in Python, so hot loops build it once."""

    def __init__(self, tensors, device=None):
        if tensors and isinstance(tensors[0], (list, tuple)):
            tensors = [g for gw in tensors for g in gw]
        self.tensors = list(tensors)          # keep the storage alive
        self.n = len(self.tensors)
        self.arr = _ptr_array(_data_ptrs(self.tensors, device))


class _DevArray:
    """Zero-copy __cuda_array_interface__ wrapper for library-owned memory."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4",
                                         "data": (ptr, False), "version": 3, "strides": None}


def torch_allgather(group=None):
    """An allgather callback over torch.distributed (gloo/CPU group)."""
    import torch
    import torch.distributed as dist

    def cb(send, recv, nbytes, _user):
        try:
            world = dist.get_world_size(group)
            src = torch.frombuffer(bytearray(C.string_at(send, nbytes)), dtype=torch.uint8)
            outs = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(outs, src, group=group)
            blob = b"".join(bytes(o.numpy().tobytes()) for o in outs)
            C.memmove(recv, blob, len(blob))
            return 0
        except Exception:  # noqa: BLE001 -- reported as CMN_ERR_BOOTSTRAP
            return 1

    return AllgatherFn(cb)


# ------------------------------------------------------------- host-only

def plan_layout(shapes):
    """cmn_plan_layout: (offsets list[T+1], L, structure hash)."""
    nd, dims = _shapes_args(shapes)
    T = len(shapes)
    off = (C.c_int64 * (T + 1))()
    L = C.c_int64()
    h = C.c_uint64()
    _check(lib().cmn_plan_layout(T, nd, dims, off, C.byref(L), C.byref(h)), "cmn_plan_layout")
    return list(off), L.value, h.value


def plan_bucket_ranges(sizes, bucket_bytes: int):
    """cmn_plan_bucket_ranges: list of (t_begin, t_end), bucket 0 = last tensors."""
    T = len(sizes)
    numel = (C.c_int64 * T)(*[int(n) for n in sizes])
    n = C.c_int()
    b = (C.c_int * T)()
    e = (C.c_int * T)()
    _check(lib().cmn_plan_bucket_ranges(T, numel, bucket_bytes, C.byref(n), b, e),
           "cmn_plan_bucket_ranges")
    return [(b[i], e[i]) for i in range(n.value)]


def plan_chunks(L: int, world: int):
    s = (C.c_int64 * world)()
    e = (C.c_int64 * world)()
    _check(lib().cmn_plan_chunks(L, world, s, e), "cmn_plan_chunks")
    return list(s), list(e)


def bootstrap_verify(rank: int, world: int, structure_hash: int, group=None) -> int:
    """Returns the cmn_status (0 = all ranks agree, 5 = mismatch)."""
    cb = torch_allgather(group)
    return lib().cmn_bootstrap_verify(rank, world, cb, None, structure_hash)


def share_fd(rank: int, world: int, fd: int, group=None) -> int:
    """cmn_share_fd: rank 0's fd, received by every rank (host-only)."""
    cb = torch_allgather(group)
    out = C.c_int(-1)
    _check(lib().cmn_share_fd(rank, world, cb, None, fd, C.byref(out)), "cmn_share_fd")
    return out.value


# -------------------------------------------------------------- communicator

class Comm:
    """One rank's communicator ("a communicator component that
    controls all inter-process communication")."""

    def __init__(self, handle: int, world: int, rank: int, simulated: bool, device: int, cb=None):
        self._h = C.c_void_p(handle)
        self.world = world
        self.rank = rank
        self.simulated = simulated
        self.device = device
        self._cb = cb          # keep the allgather callback alive
        self.T = 0
        self.shapes = []
        self._params = []

    # construction --------------------------------------------------------
    @classmethod
    def simulated_world(cls, world: int, device: int = 0) -> "Comm":
        h = C.c_void_p()
        _check(lib().cmn_init_simulated(world, device, C.byref(h)), "cmn_init_simulated")
        return cls(h.value, world, 0, True, device)

    @classmethod
    def emulated_world(cls, world: int, device: int = 0) -> "Comm":
        """cmn_init_emulated: the simulated world with its one-/two-shot
        all-reduces run as ONE cooperative launch over every rank, the
        cross-rank barriers live (include/cmn.h)."""
        h = C.c_void_p()
        _check(lib().cmn_init_emulated(world, device, C.byref(h)), "cmn_init_emulated")
        return cls(h.value, world, 0, True, device)

    @classmethod
    def init(cls, rank: int, world: int, device: int, group=None) -> "Comm":
        cb = torch_allgather(group) if world > 1 else AllgatherFn(lambda *a: 1)
        h = C.c_void_p()
        _check(lib().cmn_init(rank, world, device, cb, None, C.byref(h)), "cmn_init")
        return cls(h.value, world, rank, False, device, cb)

    def finalize(self):
        if self._h:
            lib().cmn_finalize(self._h)
            self._h = None

    def __del__(self):
        try:
            self.finalize()
        except Exception:  # noqa: BLE001
            pass

    # registration ---------------------------------------------------------
    def register_params(self, params) -> None:
        shapes = [tuple(p.shape) for p in params]
        nd, dims = _shapes_args(shapes)
        arr = _ptr_array(_data_ptrs(params, self.device))
        _check(lib().cmn_register_params(self._h, len(params), nd, dims, arr), "cmn_register_params")
        self.T = len(params)
        self.shapes = shapes
        self._params = list(params)

    def layout(self):
        off = (C.c_int64 * (self.T + 1))()
        L = C.c_int64()
        _check(lib().cmn_get_layout(self._h, off, C.byref(L)), "cmn_get_layout")
        return list(off), L.value

    # the step ---------------------------------------------------------------
    def prepare(self, grads) -> PtrTable:
        """Marshal a gradient table once (see PtrTable)."""
        return PtrTable(grads, self.device)

    def _grad_table(self, grads):
        if isinstance(grads, PtrTable):
            return grads.arr
        if self.simulated and grads and isinstance(grads[0], (list, tuple)):
            flat = [g for gw in grads for g in gw]
        else:
            flat = list(grads)
        return _ptr_array(_data_ptrs(flat, self.device))

    def allreduce_grads(self, grads, dtype="fp32", stream=None):
        _check(lib().cmn_allreduce_grads(self._h, self._grad_table(grads), _dt(dtype), _stream(stream)),
               "cmn_allreduce_grads")

    def update_momentum_sgd(self, lr: float, mu: float, stream=None):
        _check(lib().cmn_update_momentum_sgd(self._h, lr, mu, _stream(stream)), "cmn_update_momentum_sgd")

    def step(self, grads, dtype="fp32", lr=0.1, mu=0.9, stream=None):
        _check(lib().cmn_step(self._h, self._grad_table(grads), _dt(dtype), lr, mu, _stream(stream)),
               "cmn_step")

    def step_sharded(self, grads, dtype="fp32", lr=0.1, mu=0.9, stream=None):
        _check(lib().cmn_step_sharded(self._h, self._grad_table(grads), _dt(dtype), lr, mu,
                                      _stream(stream)), "cmn_step_sharded")

    def step_host(self, host_grads, host_params=None, dtype="fp32", lr=0.1, mu=0.9, stream=None):
        flat = [x for gw in host_grads for x in gw] if host_grads and isinstance(host_grads[0], (list, tuple)) \
            else list(host_grads)
        g = _ptr_array(_data_ptrs(flat, "cpu"))
        p = _ptr_array(_data_ptrs(host_params, "cpu")) if host_params is not None else None
        _check(lib().cmn_step_host(self._h, g, p, _dt(dtype), lr, mu, _stream(stream)), "cmn_step_host")

    def step_host_packed(self, host_grads_flat, host_params_flat=None, dtype="fp32", lr=0.1, mu=0.9,
                         stream=None):
        """host_grads_flat: pinned float32 tensor of L (x world, simulated) elements in the
        packed layout; host_params_flat: None or L elements receiving the new params."""
        _data_ptrs([host_grads_flat] + ([host_params_flat] if host_params_flat is not None else []), "cpu")
        hp = host_params_flat.data_ptr() if host_params_flat is not None else None
        _check(lib().cmn_step_host_packed(self._h, host_grads_flat.data_ptr(), hp, _dt(dtype), lr, mu,
                                          _stream(stream)), "cmn_step_host_packed")

    def unpack_avg_grads(self, out, stream=None):
        _check(lib().cmn_unpack_avg_grads(self._h, _ptr_array(_data_ptrs(out, self.device)), _stream(stream)),
               "cmn_unpack_avg_grads")

    def step_adam(self, grads, dtype="fp32", alpha=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, step=1,
                  stream=None):
        _check(lib().cmn_step_adam(self._h, self._grad_table(grads), _dt(dtype), alpha, beta1, beta2,
                                   eps, step, _stream(stream)), "cmn_step_adam")

    def update_adam(self, alpha, beta1, beta2, eps, step, stream=None):
        _check(lib().cmn_update_adam(self._h, alpha, beta1, beta2, eps, step, _stream(stream)),
               "cmn_update_adam")

    # buckets ------------------------------------------------------------------
    def plan_buckets(self, bucket_bytes: int) -> int:
        n = C.c_int()
        _check(lib().cmn_plan_buckets(self._h, bucket_bytes, C.byref(n)), "cmn_plan_buckets")
        return n.value

    def get_bucket(self, b: int):
        lo, hi = C.c_int(), C.c_int()
        _check(lib().cmn_get_bucket(self._h, b, C.byref(lo), C.byref(hi)), "cmn_get_bucket")
        return lo.value, hi.value

    def allreduce_bucket(self, b, grads, dtype="fp32", stream=None):
        _check(lib().cmn_allreduce_bucket(self._h, b, self._grad_table(grads), _dt(dtype),
                                          _stream(stream)), "cmn_allreduce_bucket")

    def update_bucket(self, b, lr, mu, stream=None):
        _check(lib().cmn_update_bucket(self._h, b, lr, mu, _stream(stream)), "cmn_update_bucket")

    # config / state -------------------------------------------------------------
    def set_algo(self, algo, oneshot_max_bytes: int = 0):
        a = _ALGOS[algo] if isinstance(algo, str) else int(algo)
        _check(lib().cmn_set_algo(self._h, a, oneshot_max_bytes), "cmn_set_algo")

    def set_fused_update(self, on: bool):
        """on: False/0 off, True/1/"pull" fused all-gather + update, 2/"push" also
        fuses the pack with the reduce-scatter transfer."""
        mode = {"pull": 1, "push": 2}.get(on, on) if isinstance(on, str) else int(on)
        _check(lib().cmn_set_fused_update(self._h, mode), "cmn_set_fused_update")

    def set_pipeline(self, pieces: int):
        _check(lib().cmn_set_pipeline(self._h, pieces), "cmn_set_pipeline")

    def set_ctas(self, collective_ctas: int = 0, update_ctas: int = 0):
        _check(lib().cmn_set_ctas(self._h, collective_ctas, update_ctas), "cmn_set_ctas")

    def set_stream_ctas(self, max_ctas: int = 0):
        _check(lib().cmn_set_stream_ctas(self._h, max_ctas), "cmn_set_stream_ctas")

    def set_kernel_timing(self, on: bool):
        _check(lib().cmn_set_kernel_timing(self._h, int(bool(on))), "cmn_set_kernel_timing")

    def kernel_timing(self):
        """(summed device ms, launch count) of the timed dominant-kernel launches
        since the last call; clears the record."""
        ms, n = C.c_double(), C.c_int()
        _check(lib().cmn_get_kernel_timing(self._h, C.byref(ms), C.byref(n)), "cmn_get_kernel_timing")
        return ms.value, n.value

    def set_timeout(self, ms: int):
        _check(lib().cmn_set_timeout(self._h, ms), "cmn_set_timeout")

    def momentum(self, t: int):
        """Tensor t's momentum buffer as a zero-copy torch tensor (library-owned)."""
        import torch
        p = C.c_void_p()
        _check(lib().cmn_get_momentum(self._h, t, C.byref(p)), "cmn_get_momentum")
        n = int(self._params[t].numel())
        return torch.as_tensor(_DevArray(p.value or 0, n), device=f"cuda:{self.device}").view(self.shapes[t])

    def adam_state(self, t: int):
        import torch
        m, v = C.c_void_p(), C.c_void_p()
        _check(lib().cmn_get_adam_state(self._h, t, C.byref(m), C.byref(v)), "cmn_get_adam_state")
        n = int(self._params[t].numel())
        dev = f"cuda:{self.device}"
        return (torch.as_tensor(_DevArray(m.value, n), device=dev).view(self.shapes[t]),
                torch.as_tensor(_DevArray(v.value, n), device=dev).view(self.shapes[t]))

    def copy_packed(self, rank: int, dst, stream=None):
        _check(lib().cmn_copy_packed(self._h, rank, dst.data_ptr(), _stream(stream)), "cmn_copy_packed")

    def copy_reduced(self, rank: int, dst, stream=None):
        _check(lib().cmn_copy_reduced(self._h, rank, dst.data_ptr(), _stream(stream)), "cmn_copy_reduced")

    def debug_fill_buffers(self, pattern: int = 0x7FC07FC0, stream=None):
        """cmn_debug_fill_buffers: poison the library's packed / reduced buffers
        (default: NaN as fp32 and as fp16) -- test hook."""
        _check(lib().cmn_debug_fill_buffers(self._h, C.c_uint32(pattern), _stream(stream)),
               "cmn_debug_fill_buffers")

    def poll_error(self):
        _check(lib().cmn_poll_error(self._h), "cmn_poll_error")

    @property
    def kernel_launches(self) -> int:
        return int(lib().cmn_kernel_launches(self._h))
