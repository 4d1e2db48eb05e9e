"""B200-native ChainerMN data-parallel update step (arXiv 1908.00213 §6).

The product is libcmn.so (include/cmn.h): sm_100a kernels for the
multi-tensor gradient pack/cast, the NVSwitch P2P all-reduce (one-shot /
two-shot) and the fused average + momentum-SGD update.  This package is
the thin Python binding over it.
"""
from .cmn import (ALGO_AUTO, ALGO_NCCL, ALGO_ONESHOT, ALGO_TWOSHOT, FP16, FP32, CmnError, Comm,  # noqa: F401
                  bootstrap_verify, lib, plan_chunks, plan_layout)

__all__ = ["Comm", "CmnError", "lib", "plan_layout", "plan_chunks", "bootstrap_verify",
           "FP32", "FP16", "ALGO_AUTO", "ALGO_ONESHOT", "ALGO_TWOSHOT", "ALGO_NCCL"]
