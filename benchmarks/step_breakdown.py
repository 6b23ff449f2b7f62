#!/usr/bin/env python
"""Wall-clock breakdown of the device-resident step (engine.DevicePipeline) call by call, with a
stream synchronize after every C-ABI call, next to the same step's CUDA-event kernel total."""
import ctypes as C
import sys, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from bench import build_workload
import paper_2406_04795_b200 as P
from paper_2406_04795_b200 import _cabi, engine

wl = build_workload(sys.argv[1] if len(sys.argv) > 1 else "dof6")
a = wl.arrays
checker = P.not_free_checker(wl.problem)
pipe = engine.DevicePipeline(wl.manifold, wl.cfg, wl.template, checker)
ctx, lib, n = pipe.ctx, _cabi.lib, pipe.n
seeds = torch.from_numpy(a.seeds).cuda()
for _ in range(3):
    pipe.step(seeds.data_ptr(), a.seeds.shape[0])
torch.cuda.synchronize()
for rep in range(3):
    t = [time.perf_counter()]
    def mark():
        torch.cuda.synchronize(); t.append(time.perf_counter())
    trace = C.c_void_p(); cells = C.c_void_p(); ref = C.c_void_p()
    _cabi.check(lib.pt_trace_create(ctx.handle, pipe.field, n, pipe.cfg.lattice.scale, pipe.offset.ctypes.data,
                                    pipe.lo.ctypes.data, pipe.hi.ctypes.data, (1 << 31) - 2, float(pipe.cfg.eps), C.byref(trace)))
    _cabi.check(lib.pt_trace_run(trace, C.c_void_p(seeds.data_ptr()), a.seeds.shape[0])); mark()
    st = _cabi.TraceStats(); _cabi.check(lib.pt_trace_get_stats(trace, C.byref(st)))
    pts = torch.empty((int(st.visited_edges), n), dtype=torch.float64, device="cuda")
    _cabi.check(lib.pt_trace_points(trace, C.c_void_p(pts.data_ptr()))); mark()
    _cabi.check(lib.pt_cells_from_trace(trace, C.byref(cells))); mark()
    ck = checker.device_checker
    _cabi.check(lib.pt_refine_run(ctx.handle, pipe.field, cells, n, pipe.cfg.lattice.scale, pipe.offset.ctypes.data,
                                  pipe.template.k, pipe.tv.shape[0], pipe.tv.ctypes.data, pipe.te.shape[0], pipe.te.ctypes.data,
                                  float(pipe.cfg.eps), float(pipe.eps_dedup), ck.handle, None, 0, C.byref(ref))); mark()
    lib.pt_refine_destroy(ref); lib.pt_cells_destroy(cells); lib.pt_trace_destroy(trace); mark()
    names = ["trace_run", "trace_points", "cells", "refine_run", "destroy"]
    print(rep, " | ".join(f"{nm}: {1e3 * (t[i + 1] - t[i]):.2f}" for i, nm in enumerate(names)), f"| total {1e3 * (t[-1] - t[0]):.2f} ms")
ctx.profile(True); ctx.profile_reset()
pipe.step(seeds.data_ptr(), a.seeds.shape[0])
prof = ctx.profile_dump(); ctx.profile(False)
groups = {}
for k, v in prof.items():
    g = k.split("_")[0]
    groups[g] = groups.get(g, 0.0) + v[1]
print("kernel ms by group:", {k: round(v, 2) for k, v in groups.items()}, "total", round(sum(groups.values()), 2))
# run-to-run variation per kernel
rows = []
for rep in range(6):
    ctx.profile(True); ctx.profile_reset()
    t0 = time.perf_counter()
    pipe.step(seeds.data_ptr(), a.seeds.shape[0]); torch.cuda.synchronize()
    wall = 1e3 * (time.perf_counter() - t0)
    prof = ctx.profile_dump(); ctx.profile(False)
    rows.append((wall, prof))
names = sorted(rows[0][1], key=lambda k: -rows[0][1][k][1])[:8]
print("wall", [round(r[0], 1) for r in rows])
for k in names:
    print(f"{k:24s}", [round(r[1][k][1], 2) for r in rows])
