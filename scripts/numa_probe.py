#!/usr/bin/env python
"""PCIe copy bandwidth of pinned host buffers by NUMA placement (e2e path probe).

    python scripts/numa_probe.py

The e2e step (cmn_step_host_packed) is bound by the pinned H2D / D2H copies
of 2 x 102 MB; their speed varied 1.84-2.55 ms (H2D) between boxes and runs.
This probe pins the allocating thread to each NUMA node's CPUs in turn (first
touch places the pinned pages on that node), then times H2D, D2H and both
directions at once for a 102 MB buffer.  Prints one JSON line per node plus
the GPU's own node from sysfs."""
import glob
import json
import os
import subprocess

import torch


def gpu_numa_node(dev=0):
    try:
        bus = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader", "-i", str(dev)],
                             capture_output=True, text=True, timeout=30).stdout.strip().lower()
        bus = bus[-12:] if len(bus) > 12 else bus  # 00000000:1B:00.0 -> 0000:1b:00.0
        for p in glob.glob("/sys/bus/pci/devices/*"):
            if p.lower().endswith(bus):
                return int(open(os.path.join(p, "numa_node")).read()), open(os.path.join(p, "local_cpulist")).read().strip(), bus
        return None, None, bus
    except Exception as e:  # noqa: BLE001
        return None, None, str(e)


def parse_cpulist(s):
    out = []
    for part in s.strip().split(","):
        if "-" in part:
            a, b = part.split("-")
            out += list(range(int(a), int(b) + 1))
        elif part:
            out.append(int(part))
    return out


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def main():
    L = 25557056
    dev = torch.device("cuda:0")
    node, local, bus = gpu_numa_node()
    print(json.dumps({"gpu_bus": bus, "gpu_numa_node": node, "gpu_local_cpulist": local,
                      "allowed_cpus": len(os.sched_getaffinity(0))}), flush=True)
    d_in = torch.empty(L, dtype=torch.float32, device=dev)
    d_out = torch.empty(L, dtype=torch.float32, device=dev)
    s2 = torch.cuda.Stream()
    orig = os.sched_getaffinity(0)
    nodes = sorted(glob.glob("/sys/devices/system/node/node[0-9]*"))
    for nd in nodes + ["default"]:
        if nd == "default":
            cpus, name = orig, "default"
        else:
            cpus = set(parse_cpulist(open(os.path.join(nd, "cpulist")).read())) & orig
            name = os.path.basename(nd)
            if not cpus:
                continue
        os.sched_setaffinity(0, cpus)
        h_in = torch.empty(L, dtype=torch.float32).pin_memory()
        h_out = torch.empty(L, dtype=torch.float32).pin_memory()
        h_in.fill_(1.0)
        h_out.fill_(0.0)
        os.sched_setaffinity(0, orig)
        h2d = timed(lambda: d_in.copy_(h_in, non_blocking=True))
        d2h = timed(lambda: h_out.copy_(d_out, non_blocking=True))

        def both():
            cur = torch.cuda.current_stream()
            s2.wait_stream(cur)
            d_in.copy_(h_in, non_blocking=True)
            with torch.cuda.stream(s2):
                h_out.copy_(d_out, non_blocking=True)
            cur.wait_stream(s2)
        bi = timed(both)
        print(json.dumps({"host_node": name, "cpus": len(cpus), "h2d_us": h2d, "d2h_us": d2h,
                          "both_us": bi, "h2d_gbs": 4 * L / h2d / 1e3, "d2h_gbs": 4 * L / d2h / 1e3}),
              flush=True)
        del h_in, h_out


if __name__ == "__main__":
    main()
