"""bench.py's driver contract on the GPU: N = 1 directly, and N = 2 / 8
under torchrun with one GPU per rank (skipped on a box with fewer GPUs:
ranks whose kernels spin on each other's flags are never time-sliced on one
GPU, B200_PROFILING.md): exactly one JSON line on stdout with the
contract's keys, a positive kernel count, a roofline of the dominant
kernel, the e2e number with its byte counts, clocks, and at N > 1 the
replicas bitwise equal after the timed steps."""
import json
import os
import socket
import subprocess
import sys

import pytest
from conftest import require_gpus_for_ranks

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
        "gpu_launches", "clocks")


def _check(line, n):
    d = json.loads(line)
    for k in KEYS:
        assert k in d, k
    assert d["n_gpus"] == n and d["steps"] == 4 and d["warmup"] == 3
    assert d["value"] > 0 and d["gpu_launches"] > 0
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["achieved"] > 0 and r["peak"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    return d


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_n1_contract():
    p = subprocess.run([sys.executable, "bench.py", "--steps", "4", "--warmup", "3",
                        "--min-warmup-s", "0", "--cpu-budget-s", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [x for x in p.stdout.splitlines() if x.strip()]
    assert len(lines) == 1, p.stdout
    d = _check(lines[0], 1)
    assert d["roofline"]["bound"] == "hbm" and d["cpu_baseline"]["kind"] == "oracle"
    assert d["cpu_baseline"]["cores"] == 1
    if (os.cpu_count() or 1) > 1:  # SURVEY d.5 (ii): the partitioned oracle on every core
        th = d["cpu_baseline"]["threaded"]
        assert th["cores"] == os.cpu_count() and th["value"] > 0


def test_bench_n2_torchrun_contract():
    require_gpus_for_ranks(2)
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                        str(_free_port()), "bench.py", "--gpus", "2", "--steps", "4", "--warmup", "3",
                        "--min-warmup-s", "0"],
                       cwd=ROOT, capture_output=True, text=True, timeout=1200)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [x for x in p.stdout.splitlines() if x.strip()]
    assert len(lines) == 1, p.stdout
    d = _check(lines[0], 2)
    _check_n_gt_1(d, 2)


def _check_n_gt_1(d, n):
    import bench
    assert d["details"]["replicas_bitwise_equal"] is True
    assert d["cpu_baseline"] is None           # rank 0 at N = 1 only
    assert d["config"] == bench.common_config(25557032, 161, 25557056, "fp32", n)
    r = d["roofline"]
    # the north-star quantity: the whole step's bus bytes over ms_per_step
    bus_bytes = 2 * (n - 1) / n * 4 * 25557032
    assert abs(r["achieved"] - bus_bytes / (d["ms_per_step"] * 1e-3) / 1e9) <= 1e-6 * r["achieved"]
    assert abs(r["frac"] - r["achieved"] / 770.0) < 1e-9
    assert abs(r["frac_of_nominal"] - r["achieved"] / 900.0) < 1e-9
    k = r["kernel_only"]
    # the collective kernels' own device time comes from a separate pass (time-sliced ranks on
    # one GPU make the two passes differ), so only its presence and consistency are checked
    assert k["achieved"] > 0 and abs(k["frac"] - k["achieved"] / 770.0) < 1e-9
    c = d["details"]["comparisons"]
    assert c["cmn"]["allreduce_incl_pack_us"] > 0 and c["cmn"]["allreduce_incl_pack_bus_gbs"] > 0
    for alt in ("nccl", "nvls"):          # measured, or why not (one GPU: NCCL refuses 2 ranks)
        assert "unavailable" in c[alt] or c[alt]["allreduce_incl_pack_us"] > 0
    # NVLS was first tried in isolated child processes (one GPU: multicast refused)
    pr = c["nvls"]["probe"]
    assert pr["probe"].startswith("child process") and pr["probe_s"] > 0
    assert "unavailable" in pr or pr.get("passed") is not None
    assert d["details"]["schedule_trials_us"]
    assert d["details"]["tune_budget_s"] is not None
    sw = d["details"]["config5_sweep"]          # BASELINE config 5, budget-bounded
    assert sw and sw[0]["bytes"] == 64 << 10 and all(x["cmn_us"] > 0 and x["cmn_bus_gbs"] > 0 for x in sw)
    assert all("nccl_us" in x or "nccl" in x for x in sw)


def test_bench_nvls_probe_plumbing():
    """The isolated NVLS probe's machinery (child processes with their own
    process group and CUDA context, the tolerance gate against the tree sums,
    the timings, the replica check, the collective verdict), driven with the
    two-shot P2P all-reduce standing in for the multimem kernel: every child
    passes, and because the algorithm was not NVLS the parent does not
    adopt it."""
    require_gpus_for_ranks(2)
    env = dict(os.environ, CMN_TEST_NVLS_PROBE_ALGO="twoshot")
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                        str(_free_port()), "bench.py", "--gpus", "2", "--steps", "4", "--warmup", "3",
                        "--min-warmup-s", "0", "--tune-budget-s", "1", "--sweep-budget-s", "0",
                        "--no-e2e"],
                       cwd=ROOT, capture_output=True, text=True, timeout=1200, env=env)
    tb = p.stderr.find("Traceback")
    assert p.returncode == 0, p.stderr[tb: tb + 3000] if tb >= 0 else p.stderr[-3000:]
    d = json.loads(p.stdout.strip().splitlines()[-1])
    nv = d["details"]["comparisons"]["nvls"]
    pr = nv["probe"]
    assert pr["algo"] == "twoshot" and pr["passed"] is True, pr
    assert pr["tolerance_ratio_vs_tree"] == 0.0          # the same algorithm: identical sums
    assert pr["replicas_bitwise_equal"] is True
    for k in ("allreduce_incl_pack_us", "serial_step_us", "pipelined4_step_us"):
        assert pr[k] > 0
    assert "unavailable" in nv                            # not adopted: not the NVLS algorithm
    assert not d["details"]["schedule"].startswith("nvls")


@pytest.mark.parametrize("algo", ["twoshot", "nvls"])
def test_bench_nvls_child_single_rank(algo):
    """The NVLS probe's child process (bench.py --nvls-child) on its own, one
    rank on the one GPU (no cross-rank waiting): with the two-shot kernel
    standing in it sets up, passes the tolerance gate (identical sums),
    times the all-reduce and both step schedules and checks the replica;
    with the real NVLS algorithm it reports why multicast is unavailable
    (the one-GPU boxes refuse multicast objects) -- either way exactly one
    JSON object on stdout and exit code 0."""
    env = dict(os.environ, RANK="0", WORLD_SIZE="1", LOCAL_RANK="0",
               CMN_NVLS_CHILD_INIT=f"tcp://127.0.0.1:{_free_port()}")
    if algo != "nvls":
        env["CMN_TEST_NVLS_PROBE_ALGO"] = algo
    p = subprocess.run([sys.executable, "bench.py", "--nvls-child", "--dtype", "fp32", "--gpus", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [x for x in p.stdout.splitlines() if x.strip()]
    assert len(lines) == 1, p.stdout
    r = json.loads(lines[0])
    assert r["probe"].startswith("child process") and r["algo"] == algo
    if algo == "nvls":
        assert "unavailable" in r or r.get("passed") is True, r
    else:
        assert r["passed"] is True and r["tolerance_ratio_vs_tree"] == 0.0, r
        assert r["replicas_bitwise_equal"] is True
        assert all(r[k] > 0 for k in ("allreduce_incl_pack_us", "serial_step_us", "pipelined4_step_us"))


def test_bench_n8_contract():
    """8 ranks, one GPU each (what a SCALE run at N = 8 executes): the line
    carries the same N > 1 fields; a 2 s autotune budget keeps it bounded."""
    require_gpus_for_ranks(8)
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "8", "--master-addr", "127.0.0.1", "--master-port",
                        str(_free_port()), "bench.py", "--gpus", "8", "--steps", "4", "--warmup", "3",
                        "--min-warmup-s", "0", "--tune-budget-s", "2", "--no-e2e"],
                       cwd=ROOT, capture_output=True, text=True, timeout=1800)
    tb = p.stderr.find("Traceback")
    assert p.returncode == 0, p.stderr[tb: tb + 3000] if tb >= 0 else p.stderr[-3000:]
    lines = [x for x in p.stdout.splitlines() if x.strip()]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 8 and d["e2e"] is None
    _check_n_gt_1(d, 8)


def test_reference_arm_same_config_as_gpu_arm():
    """The driver compares the two arms' config objects: identical."""
    outs = []
    for impl in ("cmn", "reference"):
        p = subprocess.run([sys.executable, "bench.py", "--impl", impl, "--steps", "4", "--warmup", "3",
                            "--min-warmup-s", "0", "--no-cpu-baseline", "--no-e2e"],
                           cwd=ROOT, capture_output=True, text=True, timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        outs.append(json.loads(p.stdout.strip().splitlines()[-1]))
    assert outs[0]["config"] == outs[1]["config"]
    assert outs[1]["steps"] == 4 and outs[1]["details"]["timed_region_s"] > 0


def _probe_parent(rank, world, port, q):
    import types

    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["CMN_TEST_NVLS_SETUP_ONLY"] = "1"      # inherited by the child processes
    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        res, adopted = bench.nvls_probe(types.SimpleNamespace(dtype="fp32"), rank, world,
                                        rank % torch.cuda.device_count(), timeout_s=240)
        q.put((rank, res, adopted))
    finally:
        dist.destroy_process_group()


def test_bench_nvls_probe_two_ranks_setup_only():
    """The isolated NVLS probe across 2 ranks up to the NVLS setup and no
    further (CMN_TEST_NVLS_SETUP_ONLY: no barrier kernel runs, so both ranks
    may share the one GPU): two parent processes (gloo) spawn their child
    processes, which rendezvous on their own port, build the communicator
    (CUDA-IPC exchange), register the ResNet-50 set and set NVLS up
    collectively -- refused on a box without a multicast fabric.  Each
    child must come back with its JSON report (the algorithm it tried and
    why it is unavailable, or that setup succeeded), and the parents must
    agree not to adopt NVLS (a setup-only probe never passes the gate)."""
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_probe_parent, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted([q.get(timeout=400) for _ in range(2)], key=lambda r: r[0])
    for p in ps:
        p.join(timeout=60)
    for rank, r, adopted in res:
        assert adopted is False
        assert r.get("algo") == "nvls", r                 # the child's own report, not a crash
        assert "unavailable" in r or r.get("setup_only") is True, r
