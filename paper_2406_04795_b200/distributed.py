"""Sharding of the hot path across GPUs (one process per GPU, torch.distributed).

    BFS trace       small traces (up to `replicate_trace_below` edges, default 2 M): run whole on every rank, no collective
                    -- a wave of the owner-hashed BFS costs about a millisecond of host-synchronised launches and collectives
                    whatever its size (measured over NCCL, benchmarks/sharded_phases.py).  Larger ones:
                    owner-hashed: rank r owns the edges whose base vertex hashes to r; per wave three collectives --
                    all_gather of the W x W count matrix, ONE all_to_all of 16-byte candidate records, all_gather of the
                    winners' tags (padded to a bound the count matrix already gives) -- admission by minimum tag on the
                    owner, global admission order from the tags (`ShardedTrace`)
    coarse cells    every rank enumerates the cell cofaces of ITS edges, then the sorted unique cell list is built by a
                    range-partitioned sample sort of the packed 64-bit cell keys: all_gather of a few samples per rank ->
                    common splitters -> all_to_all of key ranges -> local sort + unique.  Rank r ends up with the r-th
                    contiguous piece of the globally sorted list (the order contract of reference subdivision.py:141); no
                    rank ever holds all cells
    refine          rank r refines its piece (crossing sets are per cell; crossing offsets = exclusive scan over ranks)
    eps-dedup       priorities are global first-crossing indices, i.e. rank-major.  A rank's candidates lie in a slab of
                    coordinate 0 (keys sort by it first), so only points within eps of another rank's slab are exchanged
                    (ghosts).  Every rank runs the greedy dedup over own + ghost points; ghosts are then pinned to their
                    owners' verdicts and the run repeated until no verdict differs anywhere -- the greedy rule
                    (subdivision.py:195-217) has exactly one fixed point, so this is the single-GPU result
    collision       labels of the kept points stay with their rank; counts are all_reduced

The drivers are written against a small engine protocol so the exchange logic runs unchanged over NCCL with the CUDA
engine and over gloo in the CPU test-suite (tests/test_distributed_gloo.py, tests/test_sharded_trace.py).  Nothing here has
run at N > 1 on real GPUs (one GPU per box in this project): several engines on one device, gloo staging, and the real NCCL
backend on a one-rank group with every collective issued anyway (PERMATRACE_B200_FORCE_COLLECTIVES=1).
"""

from __future__ import annotations

import ctypes as C
import os

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
        # collectives run when there is somebody to talk to -- or, with PERMATRACE_B200_FORCE_COLLECTIVES=1, on a one-rank
        # group as well: the only way to drive the sharded code through the real NCCL backend on a one-GPU box
        self.collective = self.world > 1 or (self.on and os.environ.get("PERMATRACE_B200_FORCE_COLLECTIVES") == "1")
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
        if self.collective:
            self.dist.all_reduce(t, group=self.group)
        return [int(v) for v in t.tolist()]

    def _gather_rows(self, vec):
        """all_gather of equal-length 1-D tensors on the transport device into ONE [world, len] tensor (flat output buffer:
        no per-rank output list, no stack)."""
        import torch
        vec = vec.contiguous()
        out = torch.empty(self.world * vec.numel(), dtype=vec.dtype, device=vec.device)
        self.dist.all_gather_into_tensor(out, vec, group=self.group)
        return out.view(self.world, vec.numel())

    def _exchange(self, records, counts):
        """all_to_all of rows bucketed by destination rank (`counts[r]` consecutive rows go to rank r); any trailing shape."""
        import torch
        if not self.collective:
            return records
        recv_counts = self._exchange_counts(counts)
        return self._exchange_rows(records, counts, recv_counts)

    def _exchange_counts(self, counts):
        import torch
        send = torch.tensor([int(c) for c in counts], dtype=torch.int64, device=self.comm_device)
        recv = torch.zeros_like(send)
        self.dist.all_to_all_single(recv, send, group=self.group)
        return [int(v) for v in recv.tolist()]

    def _exchange_rows(self, records, counts, recv_counts):
        import torch
        out = torch.empty((sum(recv_counts),) + tuple(records.shape[1:]), dtype=records.dtype, device=self.comm_device)
        self.dist.all_to_all_single(out, self._out(records).contiguous(), output_split_sizes=recv_counts,
                                    input_split_sizes=[int(c) for c in counts], group=self.group)
        return self._back(out)

    def _gather_var(self, tensor):
        """all_gather of per-rank tensors with different leading sizes -> list of tensors."""
        import torch
        if not self.collective:
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

    def _wave_exchange(self, records, counts):
        """Candidates to their owners.  ONE all_gather of the per-destination counts gives every rank the whole W x W count
        matrix (its own receive sizes AND an upper bound for every rank's winner list), then one all_to_all of the records."""
        import torch
        if not self.collective:
            return records, [int(records.shape[0])]
        mine = torch.tensor([int(c) for c in counts], dtype=torch.int64, device=self.comm_device)
        matrix = self._gather_rows(mine).tolist()                   # matrix[src][dst]
        recv_counts = [int(matrix[src][self.rank]) for src in range(self.world)]
        received = self._exchange_rows(records, counts, recv_counts)
        return received, [sum(int(matrix[src][dst]) for src in range(self.world)) for dst in range(self.world)]

    def _wave_rank(self, tags, bounds, total_before: int, max_edges: int):
        """`rank_winners` over all ranks' winner tags without unpacking them: the lists travel padded to the largest bound
        with a sentinel that sorts behind every tag (so a padded row can be searched as it is), every rank's winner count
        rides in slot 0, and the ONE host read of the wave brings back those counts and this rank's number of live winners.
        Returns (gidx, alive, new_total, complete) like rank_winners."""
        import torch
        if not self.collective:
            return rank_winners([tags], self.rank, total_before, max_edges)
        W, k = self.world, int(tags.shape[0])
        cap = max(max(bounds), 1)
        sentinel = torch.iinfo(torch.int64).max
        padded = torch.full((cap + 1,), sentinel, dtype=torch.int64, device=self.comm_device)
        padded[0] = k
        padded[1:1 + k] = self._out(tags)
        stacked = self._back(self._gather_rows(padded))
        if k:
            below = torch.searchsorted(stacked[:, 1:].contiguous(), tags.unsqueeze(0).expand(W, k).contiguous()).sum(dim=0)
        else:
            below = torch.zeros(0, dtype=torch.int64, device=tags.device)
        gidx = below + int(total_before)
        dead = gidx >= int(max_edges)
        gidx = torch.where(dead, torch.full_like(gidx, -1), gidx)
        host = torch.cat([stacked[:, 0], (~dead).sum().reshape(1)]).tolist()
        wave_total, alive = sum(int(v) for v in host[:W]), int(host[W])
        new_total = min(int(total_before) + wave_total, int(max_edges))
        return gidx, alive, new_total, int(total_before) + wave_total <= int(max_edges)

    def run(self, seeds, max_edges: int) -> dict:
        eng = self.engine
        local_frontier, total = eng.trace_locate(seeds, self.rank, self.world)
        frontier = self._sum([local_frontier])[0]
        levels, complete = 0, total <= max_edges
        while frontier > 0 and complete:
            # per wave: all_gather(counts) + all_to_all(records) + all_gather(padded winner tags, ranked in place)
            records, counts = eng.wave_candidates()
            received, bounds = self._wave_exchange(records, counts)
            tags = eng.wave_admit(received)
            gidx, alive, new_total, complete = self._wave_rank(tags, bounds, total, max_edges)
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
    """trace -> coarse_cells -> refine(+check) sharded over the process group (see the module docstring).

    `engine` implements (tensors on `engine.tensor_device`):
        trace(seeds) -> dict(trace_edges=int, cells=int, closure_ok=bool, ...)          single-rank trace + cells
        candidates(first, count) -> (points [U, n] float64 in first-crossing order, crossing_edges int)
        dedup_label(points [M, n]) -> (kept_index int64, labels uint8)                  greedy dedup in the given order
      and, for the fully sharded path (world > 1):
        the ShardedTrace protocol, local_points()
        local_cell_keys() -> sorted unique int64 keys of the cells around THIS rank's edges (order = cell order)
        set_cells_from_keys(keys int64) -> number of distinct cells now held (sorted, deduplicated)
        dedup_mask(points [M, n] in priority order, forced int8 [M]) -> uint8 [M] kept mask (forced: 1 kept, 0 removed, -1 open)
        label(points) -> uint8 non-free mask
    An engine without `local_cell_keys` gets the replicated variant: every rank builds all cells and deduplicates the
    all_gathered candidates (kept for single-rank engines and as the reference the sharded variant is tested against).
    """

    SAMPLES_PER_RANK = 64
    MAX_PIN_ROUNDS = 64

    def __init__(self, engine, group=None, gather_result: bool = True):
        self._init_transport(engine, group)
        self.gather_result = gather_result

    # ---- sharded coarse cells: range-partitioned sample sort of the packed cell keys -------------------------
    def _range_partition(self, keys):
        """`keys`: this rank's sorted unique int64 cell keys.  Returns the keys of all ranks that fall into this rank's
        range (unsorted concatenation of sorted runs; duplicates between ranks still present)."""
        import torch
        W, k = self.world, int(keys.shape[0])
        ns = min(k, self.SAMPLES_PER_RANK * W)
        pick = torch.linspace(0, max(k - 1, 0), ns, device=keys.device).round().long() if ns else keys.new_zeros(0, dtype=torch.int64)
        pool = torch.sort(torch.cat(self._gather_var(keys[pick] if ns else keys[:0]))).values
        if pool.numel() == 0:
            return keys
        splitters = pool[(torch.arange(1, W, device=pool.device) * pool.numel()) // W]
        cut = torch.searchsorted(keys, splitters.to(keys.device))          # keys >= splitter r go right of cut[r]
        edges = [0] + [int(c) for c in cut.tolist()] + [k]
        counts = [edges[r + 1] - edges[r] for r in range(W)]
        return self._exchange(keys, counts)

    # ---- sharded eps-dedup: slab ghosts + pinning to the owners' verdicts ------------------------------------
    def _sharded_dedup(self, pts, prio_offset: int):
        """Greedy first-keeper dedup of the union of all ranks' candidates (priority = global first-crossing index,
        `prio_offset` + local position).  Returns this rank's uint8 kept mask and the number of pin rounds."""
        import torch
        eng, W, me = self.engine, self.world, self.rank
        eps = float(eng.eps_dedup)
        m, n = int(pts.shape[0]), int(pts.shape[1])
        dev = pts.device
        x0 = pts[:, 0]
        if m:
            mine = self._out(torch.stack([x0.min() - eps, x0.max() + eps]))
        else:
            mine = torch.tensor([float("inf"), float("-inf")], dtype=torch.float64, device=self.comm_device)
        spans = self._gather_rows(mine).tolist()
        # my points that may lie within eps of a point of rank r (by coordinate 0): ghosts over there
        send_idx = []
        for r in range(W):
            lo, hi = float(spans[r][0]), float(spans[r][1])
            if r == me or not m or lo > hi:
                send_idx.append(torch.zeros(0, dtype=torch.int64, device=dev))
            else:
                send_idx.append(torch.nonzero((x0 >= lo) & (x0 <= hi)).flatten())
        counts = [int(i.numel()) for i in send_idx]
        order_out = torch.cat(send_idx)
        recv_counts = self._exchange_counts(counts)
        ghost_pts = self._exchange_rows(pts[order_out], counts, recv_counts)
        g = int(ghost_pts.shape[0])
        # priorities are rank-major and the ghosts arrive bucketed by source rank, each bucket in ascending index order:
        # [ghosts of lower ranks | own points | ghosts of higher ranks] IS the priority order -- nothing to sort
        g_lo = int(sum(recv_counts[:me]))
        all_pts = torch.cat([ghost_pts[:g_lo], pts, ghost_pts[g_lo:]]) if g else pts
        forced_g = None
        rounds = 0
        while True:
            forced = torch.full((g + m,), -1, dtype=torch.int8, device=dev)
            if forced_g is not None:
                forced[:g_lo] = forced_g[:g_lo].to(torch.int8)
                forced[g_lo + m:] = forced_g[g_lo:].to(torch.int8)
            mask = eng.dedup_mask(all_pts, forced)
            own = mask[g_lo:g_lo + m]
            used = forced_g if forced_g is not None else torch.cat([mask[:g_lo], mask[g_lo + m:]])
            # the owners' verdicts on my ghosts = their masks over what they sent me, in the order it was sent
            auth = self._exchange_rows(own[order_out].to(torch.int64), counts, recv_counts)
            differ = int((used.to(torch.int64) != auth).sum().item()) if g else 0
            rounds += 1
            if self._sum([differ])[0] == 0:
                return own.to(torch.uint8), rounds
            if rounds >= self.MAX_PIN_ROUNDS:
                raise RuntimeError("sharded eps-dedup did not settle")
            forced_g = auth

    def _run_sharded(self, seeds) -> dict:
        import torch
        eng = self.engine
        info = None
        small = int(getattr(eng, "replicate_trace_below", 0))
        if small > 0 and hasattr(eng, "cell_slice_keep"):
            # Latency regime: a trace of up to `small` edges is a few dozen waves of sub-millisecond kernels, and sharding it
            # buys three collectives + five host reads per wave for nothing.  Every rank runs the same (deterministic)
            # single-device trace and cell build, capped at `small` edges, and keeps ITS contiguous range of the sorted
            # cell list; a trace that hits the cap is discarded and done again by the owner-hashed BFS below.
            cap = int(eng.max_edges)
            whole = eng.trace(seeds, max_edges=small if small < cap else None)
            if small >= cap or whole["complete"]:
                first, count = cell_slice(whole["cells"], self.rank, self.world)
                eng.cell_slice_keep(first, count)
                info = dict(whole, replicated_trace=True)
        if info is None:
            st = ShardedTrace(eng, self.group)
            info = st.run(seeds, int(eng.max_edges))
            if hasattr(eng, "local_points"):
                eng.local_points()                 # coarse-edge intersection points: each rank solves its own edges
            count = int(eng.set_cells_from_keys(self._range_partition(eng.local_cell_keys())))
        pts, crossing = eng.candidates(0, count)
        per_rank = torch.tensor([count, int(pts.shape[0]), int(crossing)], dtype=torch.int64, device=self.comm_device)
        table = [torch.zeros_like(per_rank) for _ in range(self.world)]
        self.dist.all_gather(table, per_rank, group=self.group)
        table = torch.stack(table).cpu().numpy()
        first_cell = int(table[: self.rank, 0].sum())
        prio_offset = int(table[: self.rank, 1].sum())
        kept, pin_rounds = self._sharded_dedup(pts, prio_offset)
        points = pts[kept.bool()]
        labels = eng.label(points) if hasattr(eng, "label") else torch.zeros(points.shape[0], dtype=torch.uint8)
        n_points, n_free = self._sum([int(points.shape[0]), int((labels == 0).sum().item())])
        info.update(
            cells=int(table[:, 0].sum()), slice=(first_cell, count), crossing_edges=int(table[:, 2].sum()),
            crossing_edges_local=int(crossing), candidates_local=int(pts.shape[0]), candidates=int(table[:, 1].sum()),
            crossing_offsets=np.concatenate([[0], np.cumsum(table[:, 2])[:-1]]), pin_rounds=pin_rounds,
            points_local=points, in_collision_local=labels.to(torch.bool), points_total=n_points, free_points=n_free)
        if self.gather_result:
            # rank order = global first-crossing order: the concatenation is the single-GPU result
            info["points"] = torch.cat(self._gather_var(points))
            info["in_collision"] = torch.cat(self._gather_var(labels)).to(torch.bool)
        else:
            info["points"], info["in_collision"] = points, labels.to(torch.bool)
        return info

    def run(self, seeds) -> dict:
        import torch
        dist, eng = self.dist, self.engine
        if self.collective and hasattr(eng, "local_cell_keys") and hasattr(eng, "trace_locate"):
            return self._run_sharded(seeds)
        if self.collective and hasattr(eng, "trace_locate") and getattr(eng, "shard_trace", True):
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
        if self.collective:
            counts = [torch.zeros_like(mine) for _ in range(self.world)]
            dist.all_gather(counts, mine, group=self.group)
            counts = torch.stack(counts).cpu().numpy()
            merged = torch.cat(self._gather_var(pts), dim=0)
            crossing_total = int(counts[:, 1].sum())
            crossing_offsets = np.concatenate([[0], np.cumsum(counts[:, 1])[:-1]])
        else:
            merged, crossing_total, crossing_offsets = pts, int(crossing), np.zeros(1, dtype=np.int64)
        if self.collective and hasattr(eng, "label"):
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
        # traces up to this many edges are run whole on every rank instead of owner-hashed (ShardedProof._run_sharded)
        self.replicate_trace_below = int(os.environ.get("PERMATRACE_B200_REPLICATE_TRACE_BELOW", 1 << 21))

    def _drop(self):
        lib = self._cabi.lib
        if self._cells:
            lib.pt_cells_destroy(self._cells)
        if self._trace:
            lib.pt_trace_destroy(self._trace)
        self._trace = self._cells = None

    __del__ = _drop

    def trace(self, seeds, max_edges: int | None = None) -> dict:
        """Whole trace + coarse cells on THIS device; `max_edges` caps it below the configured limit (`complete` False
        when the cap was hit: the hybrid driver then switches to the owner-hashed BFS)."""
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
            min(int(self.cfg.max_edges if max_edges is None else max_edges), (1 << 31) - 2), float(self.cfg.eps), C.byref(trace)))
        self._trace = trace
        cabi.check(lib.pt_trace_run(trace, C.c_void_p(ptr), m))
        st = cabi.TraceStats()
        cabi.check(lib.pt_trace_get_stats(trace, C.byref(st)))
        edges = int(st.visited_edges)
        if max_edges is not None and not st.complete:
            return dict(trace_edges=edges, complete=False)
        self.trace_points = torch.empty((max(edges, 1), self.n), dtype=torch.float64, device=self.tensor_device)
        if edges:
            cabi.check(lib.pt_trace_points(trace, C.c_void_p(self.trace_points.data_ptr())))
        cells = C.c_void_p()
        cabi.check(lib.pt_cells_from_trace(trace, C.byref(cells)))
        self._cells = cells
        return dict(trace_edges=edges, levels=int(st.levels), candidates_bfs=int(st.candidates),
                    vertex_evaluations=int(st.field_evaluations), closure_ok=bool(st.closure_ok), complete=bool(st.complete),
                    dropped_out_of_box=int(st.dropped_out_of_box), cells=int(lib.pt_cells_count(cells)))

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
        """(gidx [E], payload [E, n + 2] = base coordinates, step mask, sign at base) of this rank's edges; device-resident
        (the C ABI unpacks straight into the tensors)."""
        lib, cabi, torch = self._cabi.lib, self._cabi, self.torch
        st = cabi.TraceStats()
        cabi.check(lib.pt_trace_get_stats(self._trace, C.byref(st)))
        E = int(st.visited_edges)
        dev = self.tensor_device
        base = torch.zeros((E, self.n), dtype=torch.int32, device=dev)
        mask = torch.zeros(E, dtype=torch.int32, device=dev)
        sa = torch.zeros(E, dtype=torch.int8, device=dev)
        gidx = torch.zeros(E, dtype=torch.int64, device=dev)
        if E:
            cabi.check(lib.pt_trace_edges(self._trace, 0, E, C.c_void_p(base.data_ptr()), C.c_void_p(mask.data_ptr()),
                                          C.c_void_p(sa.data_ptr())))
            cabi.check(lib.pt_trace_gidx(self._trace, 0, E, C.c_void_p(gidx.data_ptr())))
        payload = torch.cat([base.to(torch.int64), mask.to(torch.int64)[:, None], sa.to(torch.int64)[:, None]], dim=1)
        return gidx, payload

    def local_cell_keys(self):
        """Sorted unique packed keys of the cells around this rank's edges (all ranks share the key window of the clamp box)."""
        lib, cabi, torch = self._cabi.lib, self._cabi, self.torch
        if self._cells:
            lib.pt_cells_destroy(self._cells)
            self._cells = None
        cells = C.c_void_p()
        cabi.check(lib.pt_cells_from_trace(self._trace, C.byref(cells)))
        self._cells = cells
        count = int(lib.pt_cells_count(cells))
        keys = torch.empty(count, dtype=torch.int64, device=self.tensor_device)
        if count:
            cabi.check(lib.pt_cells_keys(cells, 0, count, C.c_void_p(keys.data_ptr())))
        return keys

    def set_cells_from_keys(self, keys) -> int:
        """Replace the local cell list by sort + unique of `keys` (this rank's range of the global list)."""
        lib, cabi = self._cabi.lib, self._cabi
        keys = keys.contiguous()
        merged = C.c_void_p()
        cabi.check(lib.pt_cells_merge_keys(self._cells, C.c_void_p(keys.data_ptr()) if keys.shape[0] else None,
                                           keys.shape[0], C.byref(merged)))
        lib.pt_cells_destroy(self._cells)
        self._cells = merged
        return int(lib.pt_cells_count(merged))

    def cell_slice_keep(self, first: int, count: int) -> None:
        """Keep cells [first, first + count) of the (replicated) sorted cell list as this rank's range."""
        lib, cabi = self._cabi.lib, self._cabi
        sub = C.c_void_p()
        cabi.check(lib.pt_cells_slice(self._cells, first, count, C.byref(sub)))
        lib.pt_cells_destroy(self._cells)
        self._cells = sub

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
        """Sorted, deduplicated coarse cells of a merged edge list (replicated variant: every rank builds the same list)."""
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

    def dedup_mask(self, points, forced):
        """uint8 kept mask of the greedy eps-dedup over `points` (priority order) with some verdicts given (`forced`)."""
        lib, cabi, torch = self._cabi.lib, self._cabi, self.torch
        ref = C.c_void_p()
        points, forced = points.contiguous(), forced.contiguous()
        cabi.check(lib.pt_dedup_label_forced(self.ctx.handle, self.n, C.c_void_p(points.data_ptr()), points.shape[0],
                                             float(self.eps_dedup), C.c_void_p(forced.data_ptr()) if forced.shape[0] else None,
                                             None, C.byref(ref)))
        try:
            _, _, kept, _ = self._fetch(ref, False)
            mask = torch.zeros(points.shape[0], dtype=torch.uint8, device=self.tensor_device)
            mask[kept] = 1
            return mask
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

