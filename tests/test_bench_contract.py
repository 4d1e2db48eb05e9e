"""bench.py's driver contract, checked on the CPU: the reference arm (the
oracle on the host cores) prints exactly one JSON line with the contract's
keys, on the same metric / unit / config.workload as the GPU arm, and under
torchrun only rank 0 prints."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra=None, args=()):
    env = dict(os.environ)
    env.update(env_extra or {})
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "2", "--warmup", "1", *args],
                       capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr
    return [line for line in p.stdout.splitlines() if line.strip()]


def test_reference_arm_one_json_line():
    lines = _run()
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 1
    assert d["higher_is_better"] is False and d["unit"] == "us" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    import bench
    assert d["metric"] == bench.METRIC
    P, T, L = 25557032, 161, 25557056
    # the config object is identical to the GPU arm's (bench.common_config)
    assert d["config"] == bench.common_config(P, T, L, "fp32", 1)
    assert "full workload" in d["cpu_baseline"]["sample"]       # no extrapolated sample
    assert d["details"]["timed_region_s"] > 0
    blj = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert d["metric"] == blj["metric"]


def test_reference_arm_nonzero_ranks_are_silent():
    assert _run({"RANK": "1", "WORLD_SIZE": "2"}, ("--gpus", "2")) == []


def test_gpu_arm_refuses_more_ranks_than_gpus():
    """One process per GPU: bench.py never time-slices ranks whose kernels
    wait on one another on one GPU (B200_PROFILING.md) -- WORLD_SIZE larger
    than the visible GPU count (0 here) stops before any CUDA work with a
    message saying why."""
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2",
                        "--warmup", "1"], capture_output=True, text=True, env=env, timeout=300, cwd=ROOT)
    assert p.returncode != 0
    assert "2 ranks need 2 GPUs" in p.stderr
    assert not p.stdout.strip()
