"""bench.py's driver contract on the GPU: N = 1 directly and N = 2 under
torchrun (both ranks on the one test GPU): exactly one JSON line on stdout
with the contract's keys, a positive kernel count, a roofline of the
dominant kernel, the e2e number with its byte counts, clocks, and at N = 2
the replicas bitwise equal after the timed steps."""
import json
import os
import socket
import subprocess
import sys

import pytest

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
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                        str(_free_port()), "bench.py", "--gpus", "2", "--steps", "4", "--warmup", "3",
                        "--min-warmup-s", "0"],
                       cwd=ROOT, capture_output=True, text=True, timeout=1200)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [x for x in p.stdout.splitlines() if x.strip()]
    assert len(lines) == 1, p.stdout
    d = _check(lines[0], 2)
    assert d["config"]["replicas_bitwise_equal"] is True
    assert d["cpu_baseline"] is None           # rank 0 at N = 1 only
