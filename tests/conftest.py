import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: takes more than a few seconds")


def require_gpus_for_ranks(world: int):
    """Ranks whose kernels wait on one another (cross-rank barriers) need a
    GPU each: run as separate launches on one GPU nothing guarantees they run
    at the same time (B200_PROFILING.md; 2 and 4 such processes on one B200
    raised Xid 109).  On a box with fewer GPUs the test is skipped; the same
    barrier protocol runs on one GPU in tests/test_gpu_emulated.py (one
    cooperative launch over all ranks), the kernels' arithmetic in the
    simulated-world parity tests, and the host logic on CPU (gloo)."""
    import torch
    n = torch.cuda.device_count()
    if n < world:
        pytest.skip(f"{world} ranks with cross-rank barriers need {world} GPUs (this box has {n}); "
                    "never time-sliced on one GPU")


@pytest.fixture(scope="module", params=["simulated", "emulated"])
def cmn_worlds(request):
    """The binding module, once per single-GPU world kind.  In the
    "emulated" pass Comm.simulated_world builds cmn_init_emulated worlds, so
    every simulated-N test runs a second time with the one-/two-shot
    all-reduces as ONE cooperative launch over all ranks and the cross-rank
    barriers live (the schedules that have no emulated form -- fused pull /
    push, sharded -- behave as in the simulated world)."""
    from paper_1908_00213_b200 import build
    build.build()
    from paper_1908_00213_b200 import cmn as m
    m.TEST_WORLD_KIND = request.param
    if request.param == "simulated":
        yield m
        return
    saved = m.Comm.__dict__["simulated_world"]
    m.Comm.simulated_world = m.Comm.__dict__["emulated_world"]
    try:
        yield m
    finally:
        m.Comm.simulated_world = saved
        m.TEST_WORLD_KIND = "simulated"


def single_rank_only(cmn):
    """For tests that never build a simulated world (N = 1 only): run them
    in the simulated pass of conftest.cmn_worlds, skip the emulated repeat."""
    if getattr(cmn, "TEST_WORLD_KIND", "simulated") == "emulated":
        pytest.skip("N = 1 only: nothing to emulate (runs in the simulated pass)")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.lib()
    return oracle
