"""Device-resident driver of the hot path: trace -> coarse_cells -> refine(+check) with every
intermediate kept in HBM (no PermSimplex objects, no host copies of edges / cells / points).

This is what `bench.py` times for the kernel-only throughput and what a caller that only needs
the verdict (free points or none) should use; `tracer.trace` / `subdivision.refine` are the
reference-shaped wrappers around the same C ABI calls that also bring the arrays home.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _cabi

__all__ = ["DevicePipeline", "measure_fp64_peak", "measure_ex2_peak"]


def measure_fp64_peak(ctx=None) -> float:
    """FP64 FMA peak of the current device in TFLOP/s (DFMA-chain microbenchmark in the library)."""
    ctx = ctx or _cabi.context()
    return float(_cabi.lib.pt_peak_fp64(ctx.handle))


def measure_ex2_peak(ctx=None) -> float:
    """MUFU ex2 peak of the current device in T ex2/s (microbenchmark in the library)."""
    ctx = ctx or _cabi.context()
    return float(_cabi.lib.pt_peak_ex2(ctx.handle))


class DevicePipeline:
    """One proof attempt per `step`: all tables are rebuilt from empty, results stay on the device.

    With `world > 1` every rank traces (the BFS is a small share of the work) and refines the
    contiguous slice `[C*rank/world, C*(rank+1)/world)` of the sorted coarse cells; the slice
    boundaries only split work, never change which fine edges cross.
    """

    def __init__(self, manifold, cfg, template, checker, rank: int = 0, world: int = 1, device_index=None):
        self.manifold, self.cfg, self.template, self.checker = manifold, cfg, template, checker
        self.rank, self.world = rank, world
        self.ctx = _cabi.context(device_index)
        self.n = cfg.lattice.dim
        self.offset = np.asarray(cfg.lattice.offset, dtype=np.float64)
        self.lo = np.ascontiguousarray(cfg.box[0], dtype=np.float64) if cfg.box is not None else None
        self.hi = np.ascontiguousarray(cfg.box[1], dtype=np.float64) if cfg.box is not None else None
        self.tv = np.ascontiguousarray(template.vertices, dtype=np.int32)
        self.te = np.ascontiguousarray(template.edges, dtype=np.int32)
        self.eps_dedup = cfg.lattice.scale / (10.0 * template.k * template.k)
        self.field = manifold.device_field()
        self.support = manifold.support.shape[0] if hasattr(manifold, "support") else 0
        self.last_points_ptr = None

    def step(self, seeds_ptr: int, m: int) -> dict:
        lib, ctx, n = _cabi.lib, self.ctx, self.n
        work = np.zeros(6, dtype=np.int64)
        _cabi.check(lib.pt_ctx_work_counters(ctx.handle, work.ctypes.data, 1))
        trace = C.c_void_p()
        _cabi.check(lib.pt_trace_create(
            ctx.handle, self.field, n, self.cfg.lattice.scale, self.offset.ctypes.data,
            self.lo.ctypes.data if self.lo is not None else None, self.hi.ctypes.data if self.hi is not None else None,
            min(int(self.cfg.max_edges), (1 << 31) - 2), float(self.cfg.eps), C.byref(trace)))
        cells = C.c_void_p()
        sub = C.c_void_p()
        ref = C.c_void_p()
        try:
            _cabi.check(lib.pt_trace_run(trace, C.c_void_p(seeds_ptr), m))
            st = _cabi.TraceStats()
            _cabi.check(lib.pt_trace_get_stats(trace, C.byref(st)))
            edges = int(st.visited_edges)
            # coarse-edge intersection points (part of the reference's trace()); kept on the device
            import torch
            pts = torch.empty((max(edges, 1), n), dtype=torch.float64, device=f"cuda:{ctx.device}")
            if edges:
                _cabi.check(lib.pt_trace_points(trace, C.c_void_p(pts.data_ptr())))
            _cabi.check(lib.pt_cells_from_trace(trace, C.byref(cells)))
            total_cells = int(lib.pt_cells_count(cells))
            target = cells
            if self.world > 1:
                first = total_cells * self.rank // self.world
                last = total_cells * (self.rank + 1) // self.world
                _cabi.check(lib.pt_cells_slice(cells, first, last - first, C.byref(sub)))
                target = sub
            ck = getattr(self.checker, "device_checker", None)
            _cabi.check(lib.pt_refine_run(
                ctx.handle, self.field, target, n, self.cfg.lattice.scale, self.offset.ctypes.data,
                self.template.k, self.tv.shape[0], self.tv.ctypes.data, self.te.shape[0], self.te.ctypes.data,
                float(self.cfg.eps), float(self.eps_dedup), ck.handle if ck is not None else None, None, 0,
                C.byref(ref)))
            rs = _cabi.RefineStats()
            _cabi.check(lib.pt_refine_get_stats(ref, C.byref(rs)))
            _cabi.check(lib.pt_ctx_work_counters(ctx.handle, work.ctypes.data, 0))
            return {
                "trace_edges": edges, "levels": int(st.levels), "candidates": int(st.candidates),
                "vertex_evaluations": int(st.field_evaluations), "closure_ok": bool(st.closure_ok),
                "cells": total_cells, "cells_local": int(rs.cells), "crossing_edges": int(rs.crossing_edges),
                "unique_fine_edges": int(rs.unique_fine_edges), "unique_fine_vertices": int(rs.unique_fine_vertices),
                "points": int(rs.points), "free_points": int(rs.free_points), "dedup_rounds": int(rs.dedup_rounds),
                "simplices_local": (edges if self.world == 1 else 0) + int(rs.crossing_edges),
                "pair_evals_bisect": int(work[0]) * self.support, "pair_evals_eval": int(work[1]) * self.support,
                "pair_evals_fp32": int(work[2]) * self.support, "bisect_fallbacks": int(work[3]),
                "pair_evals_rest": int(work[4]) * self.support, "pair_evals_resolve": int(work[5]) * self.support,
                "pair_evals_retry": int(lib.pt_ctx_retry_evaluations(ctx.handle)) * self.support,
                "taylor_rows": int(lib.pt_ctx_taylor_rows(ctx.handle)),
                "ambiguous_signs": int(st.ambiguous_signs) + int(rs.ambiguous_signs),
            }
        finally:
            if ref:
                lib.pt_refine_destroy(ref)
            if sub:
                lib.pt_cells_destroy(sub)
            if cells:
                lib.pt_cells_destroy(cells)
            lib.pt_trace_destroy(trace)
