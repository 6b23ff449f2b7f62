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

__all__ = ["cell_slice", "owner_of_cell", "rank_winners", "ShardedTrace", "ShardedProof", "CudaEngine"]


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


def rank_winners(tag_lists, mine: int, total_before: int, max_edges: int):
    """Global admission indices of rank `mine`'s winners of one wave.

    `tag_lists[r]` is rank r's ascending tensor of winner tags.  A tag is the reference's slot id of the
    candidate (parent admission index, coface ordinal), so the wave's new edges are admitted in ascending tag
    order over ALL ranks: index = total_before + number of winners anywhere with a smaller tag.  Winners at
    or beyond `max_edges` are dead (-1) and the trace is incomplete, exactly like `_Tracer._admit`
    (reference tracer.py:239-252).  Returns (gidx int64 tensor, alive, new_total, complete)."""
    import torch
    my = tag_lists[mine]
    below = torch.zeros_like(my)
    for tags in tag_lists:
        if tags.numel():
            below += torch.searchsorted(tags, my)
    gidx = below + int(total_before)
    dead = gidx >= int(max_edges)
    gidx = torch.where(dead, torch.full_like(gidx, -1), gidx)
    wave_total = sum(int(t.numel()) for t in tag_lists)
    new_total = min(int(total_before) + wave_total, int(max_edges))
    complete = int(total_before) + wave_total <= int(max_edges)
    return gidx, int((~dead).sum().item()), new_total, complete


class _Transport:
    """Collective helpers shared by the drivers.  Buffers live on `engine.tensor_device`; when the process group
    cannot move that memory itself (gloo with CUDA tensors: CPU tests of the CUDA engine, or a box without NCCL)
    they are staged through the host for the collective only."""

    def _init_transport(self, engine, group):
        import torch
        import torch.distributed as dist
        self.engine, self.group, self.dist = engine, group, dist
        self.on = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank(group) if self.on else 0
        self.world = dist.get_world_size(group) if self.on else 1
        dev = engine.tensor_device
        staged = self.on and dist.get_backend(group) == "gloo" and torch.device(dev).type == "cuda"
        self.comm_device = torch.device("cpu") if staged else dev

    def _out(self, t):
        return t.to(self.comm_device) if t.device != self.comm_device else t

    def _back(self, t):
        dev = self.engine.tensor_device
        return t.to(dev) if t.device != dev else t

    # -- collectives (identity when there is no process group) --
    def _sum(self, values):
        import torch
        t = torch.tensor(list(values), dtype=torch.int64, device=self.comm_device)
        if self.world > 1:
            self.dist.all_reduce(t, group=self.group)
        return [int(v) for v in t.tolist()]

    def _exchange(self, records, counts):
        import torch
        if self.world == 1:
            return records
        dev = self.comm_device
        send = torch.tensor(counts, dtype=torch.int64, device=dev)
        recv = torch.zeros_like(send)
        self.dist.all_to_all_single(recv, send, group=self.group)
        recv_counts = [int(v) for v in recv.tolist()]
        out = torch.empty((sum(recv_counts), 2), dtype=torch.int64, device=dev)
        self.dist.all_to_all_single(out, self._out(records).contiguous(), output_split_sizes=recv_counts,
                                    input_split_sizes=[int(c) for c in counts], group=self.group)
        return self._back(out)

    def _gather_var(self, tensor):
        """all_gather of per-rank tensors with different leading sizes -> list of tensors."""
        import torch
        if self.world == 1:
            return [tensor]
        dev = self.comm_device
        size = torch.tensor([tensor.shape[0]], dtype=torch.int64, device=dev)
        sizes = [torch.zeros_like(size) for _ in range(self.world)]
        self.dist.all_gather(sizes, size, group=self.group)
        sizes = [int(x.item()) for x in sizes]
        padded = torch.zeros((max(max(sizes), 1),) + tuple(tensor.shape[1:]), dtype=tensor.dtype, device=dev)
        padded[: tensor.shape[0]] = self._out(tensor)
        parts = [torch.empty_like(padded) for _ in range(self.world)]
        self.dist.all_gather(parts, padded, group=self.group)
        return [self._back(parts[r][: sizes[r]]) for r in range(self.world)]


class ShardedTrace(_Transport):
    """Owner-hashed BFS over the process group (the north star's multi-GPU trace).

    Rank r owns the edges whose base lattice vertex hashes to r.  Every wave: expand the local frontier,
    all_to_all the 16-byte candidate records to their owners, admit by minimum tag on the owner, rank the
    winners' tags over all ranks (all_gather) so that every new edge gets its GLOBAL admission index,
    commit.  The union of the ranks' edges ordered by that index is the single-GPU (= reference) edge list.

    `engine` implements (records / tags are int64 torch tensors on `engine.tensor_device`):
        trace_locate(seeds, rank, world) -> (local_frontier, global_total)
        wave_candidates() -> (records [K, 2] bucketed by owner rank, counts list[int] of length world)
        wave_admit(records [M, 2]) -> ascending winner tags [V]
        wave_commit(gidx [V], alive, global_total) -> None
        trace_counters() -> dict(dropped=..., field_evaluations=..., candidates=...)   (local)
        local_edges() -> (gidx [E], payload [E, P])
    """

    def __init__(self, engine, group=None):
        self._init_transport(engine, group)

    def run(self, seeds, max_edges: int) -> dict:
        eng = self.engine
        local_frontier, total = eng.trace_locate(seeds, self.rank, self.world)
        frontier = self._sum([local_frontier])[0]
        levels, complete = 0, total <= max_edges
        while frontier > 0 and complete:
            records, counts = eng.wave_candidates()
            received = self._exchange(records, counts)
            tags = eng.wave_admit(received)
            gidx, alive, new_total, complete = rank_winners(self._gather_var(tags), self.rank, total, max_edges)
            eng.wave_commit(gidx, alive, new_total)
            frontier, total = new_total - total, new_total
            levels += 1
        c = eng.trace_counters()
        dropped, evaluations, candidates = self._sum([c["dropped"], c["field_evaluations"], c["candidates"]])
        return dict(trace_edges=total, levels=levels, complete=complete, dropped_out_of_box=dropped,
                    vertex_evaluations=evaluations, candidates_bfs=candidates,
                    closure_ok=bool(total > 0 and complete and dropped == 0))

    def gather_edges(self):
        """Every rank's edges merged in global admission order: (gidx [E], payload [E, P])."""
        import torch
        gidx, payload = self.engine.local_edges()
        all_g = torch.cat(self._gather_var(gidx))
        all_p = torch.cat(self._gather_var(payload))
        order = torch.argsort(all_g)
        return all_g[order], all_p[order]


class ShardedProof(_Transport):
    """trace -> coarse_cells -> refine(+check) with the refinement sharded over the process group.

    `engine` implements:
        trace(seeds) -> dict(trace_edges=int, cells=int, closure_ok=bool, ...)
        candidates(first, count) -> (points tensor [U, n] float64, crossing_edges int)
        dedup_label(points tensor [M, n]) -> (kept_index tensor int64, labels tensor uint8)
        tensor_device -> torch.device for the exchange buffers
    """

    def __init__(self, engine, group=None):
        self._init_transport(engine, group)

    def run(self, seeds) -> dict:
        import torch
        dist, eng = self.dist, self.engine
        if self.world > 1 and hasattr(eng, "trace_locate") and getattr(eng, "shard_trace", True):
            # owner-hashed BFS; the merged edge list (global admission order) feeds the replicated cell build
            st = ShardedTrace(eng, self.group)
            info = st.run(seeds, int(eng.max_edges))
            if hasattr(eng, "local_points"):
                eng.local_points()                 # coarse-edge intersection points: each rank solves its own edges
            _, payload = st.gather_edges()
            info["cells"] = eng.cells_from_edges(payload)
        else:
            info = dict(eng.trace(seeds))
        first, count = cell_slice(info["cells"], self.rank, self.world)
        pts, crossing = eng.candidates(first, count)
        dev = eng.tensor_device
        n = pts.shape[1]
        mine = torch.tensor([pts.shape[0], crossing], dtype=torch.int64, device=self.comm_device)
        if self.world > 1:
            counts = [torch.zeros_like(mine) for _ in range(self.world)]
            dist.all_gather(counts, mine, group=self.group)
            counts = torch.stack(counts).cpu().numpy()
            biggest = int(counts[:, 0].max())
            padded = torch.zeros((max(biggest, 1), n), dtype=torch.float64, device=self.comm_device)
            padded[: pts.shape[0]] = self._out(pts)
            gathered = [torch.empty_like(padded) for _ in range(self.world)]
            dist.all_gather(gathered, padded, group=self.group)
            merged = self._back(torch.cat([gathered[r][: int(counts[r, 0])] for r in range(self.world)], dim=0))
            crossing_total = int(counts[:, 1].sum())
            crossing_offsets = np.concatenate([[0], np.cumsum(counts[:, 1])[:-1]])
        else:
            merged, crossing_total, crossing_offsets = pts, int(crossing), np.zeros(1, dtype=np.int64)
        if self.world > 1 and hasattr(eng, "label"):
            # every rank runs the same deterministic dedup; the collision check of the kept points shards trivially
            kept, _ = eng.dedup_label(merged, label=False)
            points = merged[kept]
            lo_i, cnt_i = cell_slice(points.shape[0], self.rank, self.world)
            labels = torch.cat(self._gather_var(eng.label(points[lo_i:lo_i + cnt_i])))
        else:
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

    # ---- ShardedTrace protocol ------------------------------------------------------------------------
    @property
    def max_edges(self):
        return min(int(self.cfg.max_edges), (1 << 31) - 2)

    def trace_locate(self, seeds, rank, world):
        lib, cabi, torch = self._cabi.lib, self._cabi, self.torch
        self._drop()
        if isinstance(seeds, torch.Tensor):
            ptr, m = seeds.data_ptr(), seeds.shape[0]
        else:
            seeds = np.ascontiguousarray(seeds, dtype=np.float64)
            ptr, m = seeds.ctypes.data, seeds.shape[0]
        if self.lo is None:
            raise ValueError("the sharded trace needs TraceConfig.box (all ranks must share one key window)")
        trace = C.c_void_p()
        cabi.check(lib.pt_trace_create(self.ctx.handle, self.field, self.n, self.cfg.lattice.scale, self.offset.ctypes.data,
                                       self.lo.ctypes.data, self.hi.ctypes.data, self.max_edges, float(self.cfg.eps), C.byref(trace)))
        self._trace, self.world = trace, world
        cabi.check(lib.pt_trace_locate(trace, C.c_void_p(ptr), m))
        st = cabi.TraceStats()
        cabi.check(lib.pt_trace_get_stats(trace, C.byref(st)))
        total = int(st.visited_edges)
        cabi.check(lib.pt_trace_shard(trace, rank, world))
        cabi.check(lib.pt_trace_get_stats(trace, C.byref(st)))
        return int(st.frontier), total

    def wave_candidates(self):
        lib, cabi, torch = self._cabi.lib, self._cabi, self.torch
        counts = np.zeros(self.world, dtype=np.int64)
        cabi.check(lib.pt_trace_wave_candidates(self._trace, counts.ctypes.data))
        rec = torch.empty((int(counts.sum()), 2), dtype=torch.int64, device=self.tensor_device)
        if rec.shape[0]:
            cabi.check(lib.pt_trace_wave_fetch(self._trace, C.c_void_p(rec.data_ptr())))
        return rec, [int(c) for c in counts]

    def wave_admit(self, records):
        lib, cabi, torch = self._cabi.lib, self._cabi, self.torch
        records = records.contiguous()
        won = C.c_longlong(0)
        cabi.check(lib.pt_trace_wave_admit(self._trace, C.c_void_p(records.data_ptr()) if records.shape[0] else None,
                                           records.shape[0], C.byref(won)))
        tags = torch.empty(int(won.value), dtype=torch.int64, device=self.tensor_device)
        if tags.shape[0]:
            cabi.check(lib.pt_trace_wave_winner_tags(self._trace, C.c_void_p(tags.data_ptr())))
        return tags

    def wave_commit(self, gidx, alive, global_total):
        gidx = gidx.contiguous()
        self._cabi.check(self._cabi.lib.pt_trace_wave_commit(
            self._trace, C.c_void_p(gidx.data_ptr()) if gidx.shape[0] else None, int(alive), int(global_total)))

    def trace_counters(self):
        st = self._cabi.TraceStats()
        self._cabi.check(self._cabi.lib.pt_trace_get_stats(self._trace, C.byref(st)))
        return dict(dropped=int(st.dropped_out_of_box), field_evaluations=int(st.field_evaluations), candidates=int(st.candidates))

    def local_edges(self):
        """(gidx [E], payload [E, n + 2] = base coordinates, step mask, sign at base) of this rank's edges."""
        lib, cabi, torch = self._cabi.lib, self._cabi, self.torch
        st = cabi.TraceStats()
        cabi.check(lib.pt_trace_get_stats(self._trace, C.byref(st)))
        E = int(st.visited_edges)
        base = np.zeros((E, self.n), dtype=np.int32); mask = np.zeros(E, dtype=np.uint32); sa = np.zeros(E, dtype=np.int8)
        gidx = np.zeros(E, dtype=np.int64)
        if E:
            cabi.check(lib.pt_trace_edges(self._trace, 0, E, base.ctypes.data, mask.ctypes.data, sa.ctypes.data))
            cabi.check(lib.pt_trace_gidx(self._trace, 0, E, gidx.ctypes.data))
        payload = np.concatenate([base.astype(np.int64), mask.astype(np.int64)[:, None], sa.astype(np.int64)[:, None]], axis=1)
        return (torch.from_numpy(gidx).to(self.tensor_device), torch.from_numpy(payload).to(self.tensor_device))

    def local_points(self):
        """Intersection points of this rank's traced edges (the reference's trace() returns them), kept in HBM."""
        lib, cabi, torch = self._cabi.lib, self._cabi, self.torch
        st = cabi.TraceStats()
        cabi.check(lib.pt_trace_get_stats(self._trace, C.byref(st)))
        E = int(st.visited_edges)
        self.trace_points = torch.empty((max(E, 1), self.n), dtype=torch.float64, device=self.tensor_device)
        if E:
            cabi.check(lib.pt_trace_points(self._trace, C.c_void_p(self.trace_points.data_ptr())))
        return self.trace_points[:E]

    def cells_from_edges(self, payload) -> int:
        """Sorted, deduplicated coarse cells of the merged edge list (every rank builds the same list)."""
        lib, cabi = self._cabi.lib, self._cabi
        p = payload.cpu().numpy()
        base = np.ascontiguousarray(p[:, : self.n], dtype=np.int32)
        mask = np.ascontiguousarray(p[:, self.n], dtype=np.uint32)
        if self._cells:
            lib.pt_cells_destroy(self._cells)
            self._cells = None
        cells = C.c_void_p()
        cabi.check(lib.pt_cells_from_edges(self.ctx.handle, self.n, base.ctypes.data, mask.ctypes.data, base.shape[0], C.byref(cells)))
        self._cells = cells
        return int(lib.pt_cells_count(cells))

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

    def dedup_label(self, points, label: bool = True):
        """Greedy eps-dedup of `points` (priority order); with `label` also the collision labels of the kept points."""
        lib, cabi = self._cabi.lib, self._cabi
        ref = C.c_void_p()
        ck = getattr(self.checker, "device_checker", None) if label else None
        points = points.contiguous()
        cabi.check(lib.pt_dedup_label(self.ctx.handle, self.n, C.c_void_p(points.data_ptr()), points.shape[0],
                                      float(self.eps_dedup), ck.handle if ck is not None else None, C.byref(ref)))
        try:
            _, _, kept, labels = self._fetch(ref, True)
            return kept, labels
        finally:
            lib.pt_refine_destroy(ref)

    def label(self, points):
        """Non-free mask (outside the limits or in collision) of device points: uint8 tensor."""
        lib, cabi, torch = self._cabi.lib, self._cabi, self.torch
        points = points.contiguous()
        out = torch.zeros(points.shape[0], dtype=torch.uint8, device=self.tensor_device)
        ck = getattr(self.checker, "device_checker", None)
        if ck is not None and points.shape[0]:
            cabi.check(lib.pt_batch_check(self.ctx.handle, ck.handle, C.c_void_p(points.data_ptr()), points.shape[0],
                                          1, C.c_void_p(out.data_ptr()), None))
        return out

