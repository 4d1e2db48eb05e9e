#!/usr/bin/env python
"""Probe for the e2e step's copy plan: does splitting the 102 MB pinned
H2D / D2H transfers into pieces cost per-copy overhead, and does spreading
the pieces over several streams (copy engines) hide it?

    python scripts/pcie_streams_probe.py [--asym]    # one JSON line per variant

Variants: direction (h2d, d2h, both), pieces (1, 12, 48), streams per
direction (1, 2, 4); --asym: both directions at once with independent H2D
and D2H piece counts (1..12 each).  Each variant is timed with CUDA events around the
whole batch, median of 7 after 2 warm-ups.
"""
import json
import statistics
import sys

import torch

L = 25_557_056          # packed ResNet-50 length (fp32)


def main():
    dev = torch.device("cuda:0")
    host_in = torch.ones(L, dtype=torch.float32).pin_memory()
    host_out = torch.empty(L, dtype=torch.float32).pin_memory()
    d_in = torch.empty(L, dtype=torch.float32, device=dev)
    d_out = torch.ones(L, dtype=torch.float32, device=dev)
    main_s = torch.cuda.current_stream()
    pools = {k: [torch.cuda.Stream() for _ in range(4)] for k in ("h2d", "d2h")}

    def run(direction, pieces, streams, pieces_d2h=None):
        start = torch.cuda.Event()
        start.record(main_s)
        ends = []
        for k in (("h2d", "d2h") if direction == "both" else (direction,)):
            n = pieces_d2h if (k == "d2h" and pieces_d2h) else pieces
            bounds = [L * i // n for i in range(n + 1)]
            for j in range(streams):
                pools[k][j].wait_event(start)
            for p in range(n):
                s = pools[k][p % streams]
                a, b = bounds[p], bounds[p + 1]
                with torch.cuda.stream(s):
                    if k == "h2d":
                        d_in[a:b].copy_(host_in[a:b], non_blocking=True)
                    else:
                        host_out[a:b].copy_(d_out[a:b], non_blocking=True)
            for j in range(streams):
                e = torch.cuda.Event()
                e.record(pools[k][j])
                ends.append(e)
        for e in ends:
            main_s.wait_event(e)

    if "--asym" in sys.argv:
        plan = [("both", a, 1, b) for a in (1, 2, 3, 4, 6, 12) for b in (1, 2, 3, 4, 6, 12)]
    else:
        plan = [(d, p, st, None) for d in ("h2d", "d2h", "both") for p in (1, 12, 48)
                for st in (1, 2, 4) if st <= p]
    for direction, pieces, streams, pieces_d2h in plan:
        ts = []
        for r in range(9):
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(main_s)
            run(direction, pieces, streams, pieces_d2h)
            b.record(main_s)
            torch.cuda.synchronize()
            if r >= 2:
                ts.append(a.elapsed_time(b) * 1e3)
        us = statistics.median(ts)
        nbytes = 4 * L * (2 if direction == "both" else 1)
        print(json.dumps({"direction": direction, "pieces": pieces, "streams": streams,
                          "pieces_d2h": pieces_d2h if pieces_d2h else pieces,
                          "us": round(us, 1), "gbs": round(nbytes / us / 1e3, 1)}), flush=True)


if __name__ == "__main__":
    main()
