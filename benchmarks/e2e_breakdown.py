#!/usr/bin/env python
"""Wall-clock breakdown of one end-to-end step through the public API (host buffers)."""
import sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from bench import build_workload
import paper_2406_04795_b200 as P

wl = build_workload(sys.argv[1] if len(sys.argv) > 1 else "dof6")
a = wl.arrays
checker = P.not_free_checker(wl.problem)
scale, gain, lo, hi = a.barrier
for rep in range(4):
    t = [time.perf_counter()]
    manifold = P.KernelClassifierManifold(a.support, a.weights, a.gamma, a.bias, barrier=P.BoxBarrier(lo, hi, scale, gain))
    manifold.device_field(); t.append(time.perf_counter())
    res = P.trace(a.seeds, manifold, wl.cfg); t.append(time.perf_counter())
    cells = P.coarse_cells(res); t.append(time.perf_counter())
    ref = P.refine(cells, wl.template, manifold, checker, wl.cfg); t.append(time.perf_counter())
    names = ["field upload", "trace(+points D2H)", "coarse_cells", "refine(+points/labels D2H)"]
    print(rep, " | ".join(f"{n}: {1e3 * (t[i + 1] - t[i]):.1f} ms" for i, n in enumerate(names)), f"| total {1e3 * (t[-1] - t[0]):.1f} ms")
