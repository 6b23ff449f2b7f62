"""Sharding of the hot path across GPUs (one process per GPU, torch.distributed).

What shards: refinement and collision checking are embarrassingly parallel
over the sorted coarse cells, so rank r takes the contiguous slice [C*r/W, C*(r+1)/W).  Every rank
traces (the BFS is ~1 % of a proof and launch-latency bound at benchmark sizes; the owner-hashed
all-to-all BFS of the north star only pays once a trace no longer fits one GPU).  The only exchange
is the merge of the per-slice root-solved points before the order-dependent eps-dedup:

    1. all_gather(crossing count, candidate count)     -> global crossing-index offsets per rank
    2. all_gather(padded candidate points)             -> concatenation in rank order is already in
                                                          global first-crossing order
    3. every rank runs the same greedy eps-dedup + collision labelling on the merged list

The driver is written against a small engine protocol so the exchange logic runs unchanged over
NCCL with the CUDA engine and over gloo in the CPU test-suite (tests/test_distributed_gloo.py).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

__all__ = ["cell_slice", "owner_of_cell", "ShardedProof", "CudaEngine"]


def cell_slice(total: int, rank: int, world: int) -> tuple[int, int]:
    """(first, count) of rank's contiguous slice; slices tile [0, total) in rank order."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    first = total * rank // world
    last = total * (rank + 1) // world
    return first, last - first


def owner_of_cell(base, world: int) -> np.ndarray:
    """Owner rank of lattice cells by a hash of their integer base (the north star's ownership rule;
    same mixer as the device hash tables, csrc/pt_common.cuh pt_mix)."""
    base = np.atleast_2d(np.asarray(base, dtype=np.int64)).astype(np.uint64)
    h = np.full(base.shape[0], 0x9E3779B97F4A7C15, dtype=np.uint64)
    with np.errstate(over="ignore"):
        for d in range(base.shape[1]):
            x = h ^ base[:, d]
            x ^= x >> np.uint64(33)
            x *= np.uint64(0xFF51AFD7ED558CCD)
            x ^= x >> np.uint64(33)
            x *= np.uint64(0xC4CEB9FE1A85EC53)
            x ^= x >> np.uint64(33)
            h = x
    return (h % np.uint64(world)).astype(np.int64)


class ShardedProof:
    """trace -> coarse_cells -> refine(+check) with the refinement sharded over the process group.

    `engine` implements:
        trace(seeds) -> dict(trace_edges=int, cells=int, closure_ok=bool, ...)
        candidates(first, count) -> (points tensor [U, n] float64, crossing_edges int)
        dedup_label(points tensor [M, n]) -> (kept_index tensor int64, labels tensor uint8)
        tensor_device -> torch.device for the exchange buffers
    """

    def __init__(self, engine, group=None):
        import torch.distributed as dist
        self.engine = engine
        self.group = group
        self.dist = dist
        self.on = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank(group) if self.on else 0
        self.world = dist.get_world_size(group) if self.on else 1

    def run(self, seeds) -> dict:
        import torch
        dist, eng = self.dist, self.engine
        info = dict(eng.trace(seeds))
        first, count = cell_slice(info["cells"], self.rank, self.world)
        pts, crossing = eng.candidates(first, count)
        dev = eng.tensor_device
        n = pts.shape[1]
        mine = torch.tensor([pts.shape[0], crossing], dtype=torch.int64, device=dev)
        if self.world > 1:
            counts = [torch.zeros_like(mine) for _ in range(self.world)]
            dist.all_gather(counts, mine, group=self.group)
            counts = torch.stack(counts).cpu().numpy()
            biggest = int(counts[:, 0].max())
            padded = torch.zeros((max(biggest, 1), n), dtype=torch.float64, device=dev)
            padded[: pts.shape[0]] = pts
            gathered = [torch.empty_like(padded) for _ in range(self.world)]
            dist.all_gather(gathered, padded, group=self.group)
            merged = torch.cat([gathered[r][: int(counts[r, 0])] for r in range(self.world)], dim=0)
            crossing_total = int(counts[:, 1].sum())
            crossing_offsets = np.concatenate([[0], np.cumsum(counts[:, 1])[:-1]])
        else:
            merged, crossing_total, crossing_offsets = pts, int(crossing), np.zeros(1, dtype=np.int64)
        kept, labels = eng.dedup_label(merged)
        points = merged[kept]
        info.update(
            crossing_edges=crossing_total, crossing_edges_local=int(crossing), candidates_local=int(pts.shape[0]),
            candidates=int(merged.shape[0]), points=points, in_collision=labels.to(torch.bool),
            free_points=int((labels == 0).sum().item()), crossing_offsets=crossing_offsets, slice=(first, count),
        )
        return info


class CudaEngine:
    """The engine protocol over libpermatrace_b200.so; every array stays in HBM (torch CUDA tensors
    wrap the exchange buffers so NCCL can move them)."""

    def __init__(self, manifold, cfg, template, checker, device_index=None):
        import torch
        from . import _cabi
        self._cabi, self.torch = _cabi, torch
        self.manifold, self.cfg, self.template, self.checker = manifold, cfg, template, checker
        self.ctx = _cabi.context(device_index)
        self.tensor_device = torch.device("cuda", self.ctx.device)
        self.n = cfg.lattice.dim
        self.offset = np.asarray(cfg.lattice.offset, dtype=np.float64)
        self.lo = np.ascontiguousarray(cfg.box[0], dtype=np.float64) if cfg.box is not None else None
        self.hi = np.ascontiguousarray(cfg.box[1], dtype=np.float64) if cfg.box is not None else None
        self.tv = np.ascontiguousarray(template.vertices, dtype=np.int32)
        self.te = np.ascontiguousarray(template.edges, dtype=np.int32)
        self.eps_dedup = cfg.lattice.scale / (10.0 * template.k * template.k)
        self.field = manifold.device_field()
        self._trace = self._cells = None

    def _drop(self):
        lib = self._cabi.lib
        if self._cells:
            lib.pt_cells_destroy(self._cells)
        if self._trace:
            lib.pt_trace_destroy(self._trace)
        self._trace = self._cells = None

    __del__ = _drop

    def trace(self, seeds) -> dict:
        lib, cabi = self._cabi.lib, self._cabi
        self._drop()
        torch = self.torch
        if isinstance(seeds, torch.Tensor):
            ptr, m = seeds.data_ptr(), seeds.shape[0]
        else:
            seeds = np.ascontiguousarray(seeds, dtype=np.float64)
            ptr, m = seeds.ctypes.data, seeds.shape[0]
        trace = C.c_void_p()
        cabi.check(lib.pt_trace_create(
            self.ctx.handle, self.field, self.n, self.cfg.lattice.scale, self.offset.ctypes.data,
            self.lo.ctypes.data if self.lo is not None else None, self.hi.ctypes.data if self.hi is not None else None,
            min(int(self.cfg.max_edges), (1 << 31) - 2), float(self.cfg.eps), C.byref(trace)))
        self._trace = trace
        cabi.check(lib.pt_trace_run(trace, C.c_void_p(ptr), m))
        st = cabi.TraceStats()
        cabi.check(lib.pt_trace_get_stats(trace, C.byref(st)))
        edges = int(st.visited_edges)
        self.trace_points = torch.empty((max(edges, 1), self.n), dtype=torch.float64, device=self.tensor_device)
        if edges:
            cabi.check(lib.pt_trace_points(trace, C.c_void_p(self.trace_points.data_ptr())))
        cells = C.c_void_p()
        cabi.check(lib.pt_cells_from_trace(trace, C.byref(cells)))
        self._cells = cells
        return dict(trace_edges=edges, levels=int(st.levels), candidates_bfs=int(st.candidates),
                    vertex_evaluations=int(st.field_evaluations), closure_ok=bool(st.closure_ok),
                    cells=int(lib.pt_cells_count(cells)))

    def _fetch(self, ref, with_labels):
        lib, cabi, torch = self._cabi.lib, self._cabi, self.torch
        st = cabi.RefineStats()
        cabi.check(lib.pt_refine_get_stats(ref, C.byref(st)))
        total = int(st.points)
        pts = torch.empty((total, self.n), dtype=torch.float64, device=self.tensor_device)
        tags = torch.empty(total, dtype=torch.int64, device=self.tensor_device)
        labels = torch.zeros(total, dtype=torch.uint8, device=self.tensor_device)
        if total:
            cabi.check(lib.pt_refine_points(ref, C.c_void_p(pts.data_ptr()),
                                            C.c_void_p(labels.data_ptr()) if with_labels else None,
                                            C.c_void_p(tags.data_ptr())))
        return st, pts, tags, labels

    def candidates(self, first: int, count: int):
        lib, cabi = self._cabi.lib, self._cabi
        sub, ref = C.c_void_p(), C.c_void_p()
        try:
            cabi.check(lib.pt_cells_slice(self._cells, first, count, C.byref(sub)))
            cabi.check(lib.pt_refine_candidates(
                self.ctx.handle, self.field, sub, self.n, self.cfg.lattice.scale, self.offset.ctypes.data,
                self.template.k, self.tv.shape[0], self.tv.ctypes.data, self.te.shape[0], self.te.ctypes.data,
                float(self.cfg.eps), C.byref(ref)))
            st, pts, _, _ = self._fetch(ref, False)
            self.last_refine_stats = {name: int(getattr(st, name)) for name, _ in cabi.RefineStats._fields_}
            return pts, int(st.crossing_edges)
        finally:
            if ref:
                lib.pt_refine_destroy(ref)
            if sub:
                lib.pt_cells_destroy(sub)

    def dedup_label(self, points):
        lib, cabi = self._cabi.lib, self._cabi
        ref = C.c_void_p()
        ck = getattr(self.checker, "device_checker", None)
        points = points.contiguous()
        cabi.check(lib.pt_dedup_label(self.ctx.handle, self.n, C.c_void_p(points.data_ptr()), points.shape[0],
                                      float(self.eps_dedup), ck.handle if ck is not None else None, C.byref(ref)))
        try:
            _, _, kept, labels = self._fetch(ref, True)
            return kept, labels
        finally:
            lib.pt_refine_destroy(ref)
