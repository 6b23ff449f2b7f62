#!/usr/bin/env python
"""BFS-only throughput of the tracer on an analytic sphere (isolates the hash / frontier kernels from
field evaluation, like the reference's `cli bench` twin, cli.py:297).  Prints one JSON line per lambda.

    python benchmarks/bfs_scaling.py --dim 6 --lambdas 0.25 0.125
"""
import argparse
import ctypes as C
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

ALGO_BYTES = {4: 0.74e3, 5: 1.21e3, 6: 1.92e3}   # SURVEY.md section 8d, bytes per traced edge


def main():
    import torch
    import paper_2406_04795_b200 as P
    from paper_2406_04795_b200 import _cabi
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=6)
    ap.add_argument("--lambdas", type=float, nargs="+", default=[0.25, 0.125])
    ap.add_argument("--radius", type=float, default=0.8)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    peaks = {}
    try:
        peaks = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text())
    except OSError:
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    ctx = _cabi.context()
    lib = _cabi.lib
    n = args.dim
    field = P.SphereManifold(np.zeros(n), args.radius)
    seeds = torch.from_numpy(field.seed_point()[None, :].copy()).cuda()
    offset = np.zeros(n)
    for lam in args.lambdas:
        best = None
        for rep in range(args.reps):
            tr = C.c_void_p()
            _cabi.check(lib.pt_trace_create(ctx.handle, field.device_field(), n, lam, offset.ctypes.data, None, None,
                                            (1 << 31) - 2, 1e-9, C.byref(tr)))
            torch.cuda.synchronize()
            ctx.profile(True); ctx.profile_reset()
            t0 = time.perf_counter()
            _cabi.check(lib.pt_trace_run(tr, C.c_void_p(seeds.data_ptr()), 1))
            ctx.synchronize()
            dt = time.perf_counter() - t0
            prof = ctx.profile_dump(); ctx.profile(False)
            st = _cabi.TraceStats()
            _cabi.check(lib.pt_trace_get_stats(tr, C.byref(st)))
            lib.pt_trace_destroy(tr)
            wave_ms = sum(v[1] for k, v in prof.items() if k.startswith("trace_wave") or k == "table_rehash")
            row = {"dim": n, "lambda": lam, "edges": int(st.visited_edges), "levels": int(st.levels),
                   "candidates": int(st.candidates), "vertex_evaluations": int(st.field_evaluations),
                   "closure_ok": bool(st.closure_ok), "seconds": dt, "edges_per_s": st.visited_edges / dt,
                   "candidates_per_s": st.candidates / dt, "wave_kernel_ms": wave_ms,
                   "table_capacity": int(st.table_capacity),
                   "algorithmic_GBps": st.visited_edges * ALGO_BYTES.get(n, 0.0) / dt / 1e9,
                   "algorithmic_GBps_wave_kernels": st.visited_edges * ALGO_BYTES.get(n, 0.0) / (wave_ms * 1e-3) / 1e9 if wave_ms else None,
                   "hbm_peak_GBps": hbm,
                   "kernels_ms": {k: round(v[1], 3) for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])[:8]}}
            if best is None or row["seconds"] < best["seconds"]:
                best = row
        best["hbm_frac_wave_kernels"] = (best["algorithmic_GBps_wave_kernels"] or 0.0) / hbm
        print(json.dumps(best), flush=True)


if __name__ == "__main__":
    main()
