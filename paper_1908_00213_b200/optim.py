"""multi_node_optimizer on top of the C ABI (Fig. 4).

"multi_node_optimizer ... wraps the normal optimizer and exchanges the
gradient across processes using the all-reduce operation before optimizing
the model.  It behaves identically as the original optimizer except for the
communication."  Here the wrapped optimizer is momentum SGD (or Adam), and
exchange + update are cmn_* calls: this module is bookkeeping only (pointer
tables, backward hooks, re-registration); every arithmetic step runs in
libcmn's kernels.

Define-by-Run compatibility: "model structures are
identical between workers merely in a single iteration ... model structure
can be changed at any iteration dynamically".  step() compares the current
parameter set with the registered one and re-registers (a collective call,
so every rank re-registers in the same iteration) when it changed; the
registration-time structure check turns a cross-rank divergence into
CMN_ERR_MISMATCH instead of a hang.

Overlap: with bucket_bytes set, a post-accumulate-grad
hook counts ready gradients per bucket (buckets are reverse-order contiguous
tensor ranges) and launches cmn_allreduce_bucket on a communication stream
as soon as a bucket is complete, while backward keeps running; step() then
waits and applies cmn_update_bucket per bucket.  Buckets assume ONE backward
per step(); gradient-accumulation micro-batches run under no_sync() (their
hooks launch nothing, the last backward outside it does), and a second
backward that would re-launch a bucket before step() raises instead of
silently all-reducing a partial gradient.  Bucketed overlap is momentum-SGD
only (the bucket update is cmn_update_bucket); optimizer="adam" with
bucket_bytes is refused.
"""
from __future__ import annotations

import contextlib

import torch

from .cmn import Comm, PtrTable


class MultiNodeOptimizer:
    def __init__(self, params, comm: Comm, lr: float = 0.1, momentum: float = 0.9,
                 dtype: str = "fp32", bucket_bytes: int | None = None, optimizer: str = "momentum_sgd",
                 adam=(1e-3, 0.9, 0.999, 1e-8), stream_ctas: int = 0):
        if bucket_bytes and optimizer != "momentum_sgd":
            raise ValueError("bucketed overlap (bucket_bytes) applies momentum SGD per bucket; "
                             f"optimizer={optimizer!r} is not supported with it")
        if optimizer not in ("momentum_sgd", "adam"):
            raise ValueError(f"unknown optimizer {optimizer!r}")
        self.comm = comm
        # overlap: cap the pack/update grids so they share SMs with the
        # backward instead of taking every free slot (cmn_set_stream_ctas;
        # 64 measured best on one B200, profiles/r1_overlap_sweep.jsonl)
        comm.set_stream_ctas(stream_ctas)
        self.lr, self.mu, self.dtype = lr, momentum, dtype
        self.bucket_bytes = bucket_bytes
        self.optimizer = optimizer
        self.adam = adam
        self.t = 0
        self.registrations = 0
        self._hooks = []
        self._stream = None
        self._launched = set()
        self._no_sync = False
        self._table, self._table_key = None, None
        self._setup(list(params))

    # -------------------------------------------------------------- structure
    def _setup(self, params):
        for h in self._hooks:
            h.remove()
        self._hooks = []
        self.params = params
        self.comm.register_params(params)
        self.registrations += 1
        self.t = 0
        self._sig = [(id(p), tuple(p.shape)) for p in params]
        # bucket indices of the old plan mean nothing under the new one
        self._launched = set()
        self._pending = []
        self.buckets = []
        if self.bucket_bytes:
            nb = self.comm.plan_buckets(self.bucket_bytes)
            self.buckets = [self.comm.get_bucket(b) for b in range(nb)]
            self._bucket_of = {}
            for b, (lo, hi) in enumerate(self.buckets):
                for t in range(lo, hi):
                    self._bucket_of[t] = b
            self._pending = [hi - lo for lo, hi in self.buckets]
            if self._stream is None:
                self._stream = torch.cuda.Stream(priority=-1)
            for t, p in enumerate(params):
                self._hooks.append(p.register_post_accumulate_grad_hook(self._make_hook(t)))

    def maybe_reregister(self, params) -> bool:
        params = list(params)
        sig = [(id(p), tuple(p.shape)) for p in params]
        if sig != self._sig:
            self._setup(params)
            return True
        return False

    # ----------------------------------------------------------------- overlap
    @contextlib.contextmanager
    def no_sync(self):
        """Gradient accumulation: backwards inside launch no bucket
        all-reduce; the step's last backward (outside) does."""
        prev, self._no_sync = self._no_sync, True
        try:
            yield
        finally:
            self._no_sync = prev

    def _make_hook(self, t):
        def hook(_p):
            if self._no_sync:
                return
            b = self._bucket_of[t]
            if b in self._launched:
                raise RuntimeError(
                    "multi_node_optimizer: a second backward before step() would all-reduce a "
                    "bucket twice; run accumulation micro-batches under no_sync()")
            self._pending[b] -= 1
            if self._pending[b] == 0:
                lo, hi = self.buckets[b]
                if all(q.grad is not None for q in self.params[lo:hi]):
                    ev = torch.cuda.Event()
                    ev.record(torch.cuda.current_stream())
                    self._stream.wait_event(ev)
                    self.comm.allreduce_bucket(b, self._grad_table(), self.dtype, self._stream)
                    self._launched.add(b)
        return hook

    def _grad_table(self) -> PtrTable:
        # Only the bucket's own grads are read; others may be missing yet, so
        # absent grads point at the parameter (never dereferenced).  The
        # marshalled table is reused while the gradient storage stays put
        # (persistent .grad buffers, the usual case between zero_grad()s
        # that keep them).
        ts = [p.grad if p.grad is not None else p for p in self.params]
        key = tuple(t.data_ptr() for t in ts)
        if key != self._table_key:
            self._table, self._table_key = PtrTable(ts, self.comm.device), key
            # the pointed-to storage is kept alive by the parameters' .grad
            # (the key matched it); holding the tensors here would pin old
            # gradients across zero_grad(set_to_none)
            self._table.tensors = []
        return self._table

    # -------------------------------------------------------------------- step
    def step(self, params=None):
        if params is not None:
            self.maybe_reregister(params)
        if any(p.grad is None for p in self.params):
            raise RuntimeError("multi_node_optimizer: a registered parameter has no gradient")
        cur = torch.cuda.current_stream()
        if self.buckets:
            table = None
            for b in range(len(self.buckets)):
                if b not in self._launched:          # hook did not fire (e.g. no backward hooks)
                    if table is None:
                        table = self._grad_table()
                    ev = torch.cuda.Event()
                    ev.record(cur)
                    self._stream.wait_event(ev)
                    self.comm.allreduce_bucket(b, table, self.dtype, self._stream)
            cur.wait_stream(self._stream)
            for b in range(len(self.buckets)):
                self.comm.update_bucket(b, self.lr, self.mu, cur)
            self._launched.clear()
            self._pending = [hi - lo for lo, hi in self.buckets]
        elif self.optimizer == "adam":
            self.t += 1
            a, b1, b2, eps = self.adam
            self.comm.step_adam(self._grad_table(), self.dtype, a, b1, b2, eps, self.t)
        else:
            self.comm.step(self._grad_table(), self.dtype, self.lr, self.mu)

    def zero_grad(self):
        for p in self.params:
            p.grad = None


def create_multi_node_optimizer(params, comm: Comm, **kw) -> MultiNodeOptimizer:
    """The paper's create_multi_node_optimizer(optimizer, comm)."""
    return MultiNodeOptimizer(params, comm, **kw)
