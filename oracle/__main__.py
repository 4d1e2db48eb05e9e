"""Oracle CLI (test infrastructure): run / time the plain-C oracle on a
seeded synthetic workload.

    python -m oracle --config {mlp,r50} --workers N --dtype {fp32,fp16} \\
        [--steps K] [--seed S] [--lr 0.1] [--mu 0.9] [--set random] [--time] [--dump DIR]
        [--threads T]

Prints one JSON line: the configuration, per-step wall time (generation
excluded; single thread, or with --threads T > 1 the elementwise partition of
SURVEY §8(d) d.5 (ii), oracle.step_threaded, bit-identical w and v) and
checksums of w and v; --dump writes the reduced buffer, w and v of the last
step as .npy files (single thread only).
"""
import argparse
import json
import os
import platform
import time

import numpy as np

import oracle
import synth


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or platform.machine()


def main():
    ap = argparse.ArgumentParser(prog="python -m oracle")
    ap.add_argument("--config", default="mlp", choices=sorted(synth.WORKLOADS))
    ap.add_argument("--workers", type=int, default=2)
    ap.add_argument("--dtype", default="fp32", choices=["fp32", "fp16"])
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--seed", type=int, default=synth.BASE_SEED)
    ap.add_argument("--lr", type=float, default=0.1)
    ap.add_argument("--mu", type=float, default=0.9)
    ap.add_argument("--set", default="random", choices=sorted(synth.SET_IDS))
    ap.add_argument("--time", action="store_true")
    ap.add_argument("--dump", default=None)
    ap.add_argument("--threads", type=int, default=1, help="0 = all host cores")
    a = ap.parse_args()
    threads = a.threads or os.cpu_count() or 1
    if a.dump and threads > 1:
        ap.error("--dump needs the single-threaded step (the partition has no global reduced buffer)")
    shapes = synth.WORKLOADS[a.config]()
    w = synth.params(shapes, seed=a.seed, value_set="integer" if a.set == "integer" else "random")
    v = [np.zeros_like(x) for x in w]
    times = []
    res = None
    for s in range(a.steps):
        g = synth.grads(shapes, workers=a.workers, seed=a.seed, step=s, value_set=a.set)
        t0 = time.perf_counter()
        if threads > 1:
            oracle.step_threaded(g, w, v, a.lr, a.mu, a.dtype, threads=threads)
        else:
            res = oracle.step(g, w, v, a.lr, a.mu, a.dtype)
        times.append(time.perf_counter() - t0)
    out = {"config": a.config, "workers": a.workers, "dtype": a.dtype, "steps": a.steps, "set": a.set,
           "params": int(sum(x.size for x in w)), "threads": threads, "cpu": cpu_model(), "nproc": os.cpu_count(),
           "w_checksum": float(np.sum([np.sum(x, dtype=np.float64) for x in w])),
           "v_checksum": float(np.sum([np.sum(x, dtype=np.float64) for x in v]))}
    if a.time:
        out["step_ms"] = [t * 1e3 for t in times]
        out["step_ms_median"] = float(np.median(times) * 1e3)
    if a.dump:
        os.makedirs(a.dump, exist_ok=True)
        np.save(os.path.join(a.dump, "reduced.npy"), res["reduced"])
        np.save(os.path.join(a.dump, "w.npy"), np.concatenate([x.reshape(-1) for x in w]))
        np.save(os.path.join(a.dump, "v.npy"), np.concatenate([x.reshape(-1) for x in v]))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
