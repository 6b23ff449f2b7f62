"""Manifold tracing over the permutahedral lattice, executed as batched BFS waves on the B200.

Public names follow ``permatrace/tracer.py:24-36``.  `trace` drives ``pt_trace_run`` (locate ->
waves of probe / evaluate / partner / admit kernels, ``csrc/pt_trace.cu``) and returns a
`TraceResult` whose `edges` and `adjacency` are materialised lazily from the device arrays, in
exactly the reference's admission order (slot order = frontier index, then coface ordinal).

Semantics kept from the reference: sign convention F>0 -> +1 else -1 (tracer.py:209); partner rule
(tracer.py:343-347); inclusive box clamp in lattice units with a dropped counter
(tracer.py:187-193, :351-353); `max_edges` cap -> `complete=False` (tracer.py:243-245);
`closure_ok = edges and complete and dropped == 0` (tracer.py:399).
"""

from __future__ import annotations

import ctypes as C
from collections.abc import Sequence
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import _cabi
from .lattice import LatticeConfig, PermSimplex, edges_from_arrays, edges_to_arrays

__all__ = [
    "TraceConfig", "Frontier", "TraceStats", "StageStat", "TraceResult", "CapacityError",
    "locate_edges", "expand_frontier", "trace", "write_edgemesh", "read_edgemesh",
]

_STAGE_NAMES = ("locate_cells", "cell_edges", "edge_cofaces", "coface_partner")


class CapacityError(RuntimeError):
    """A stage produced more outputs than its preallocation bound."""


@dataclass(frozen=True)
class TraceConfig:
    """Tracing parameters: lattice, optional clamp box, budget, parallelism (tracer.py:43-59).

    `workers` is accepted for signature compatibility; results never depended on it in the
    reference and the device path ignores it.
    """

    lattice: LatticeConfig
    box: tuple[tuple[float, ...], tuple[float, ...]] | None = None
    max_edges: int = 10_000_000
    workers: int = 1
    eps: float = 1e-9

    def __post_init__(self):
        if self.max_edges < 1:
            raise ValueError("max_edges must be positive")
        if self.workers < 1:
            raise ValueError("workers must be positive")
        if self.eps <= 0:
            raise ValueError("eps must be positive")


@dataclass(frozen=True)
class Frontier:
    """Edges admitted at one BFS level, plus the producing stage's capacity."""

    edges: tuple[PermSimplex, ...]
    capacity: int
    signs: tuple[tuple[int, int], ...] | None = field(default=None, repr=False)

    def __len__(self):
        return len(self.edges)


@dataclass
class StageStat:
    name: str
    level: int
    items: int
    capacity: int
    produced: int


@dataclass
class TraceStats:
    """Counters for one trace; field_evaluations counts lattice vertex signs."""

    levels: int = 0
    seeds: int = 0
    visited_edges: int = 0
    field_evaluations: int = 0
    dropped_out_of_box: int = 0
    two_edge_violations: int = 0
    complete: bool = True
    closure_ok: bool = False
    polyline_closed: bool | None = None
    stages: list[StageStat] = field(default_factory=list)
    # not in the reference: evaluated vertices with |F| < 1e-12*(sum|w|+|bias|), the reference's own cross-backend
    # tolerance on the kernel sum (pkg/tests/test_backends.py:81-93); only such a vertex can change the traced set
    ambiguous_signs: int = 0


class _TraceHandle:
    """Owns a pt_trace and keeps the manifold (whose pt_field it references) alive."""

    def __init__(self, manifold, cfg: TraceConfig):
        n = cfg.lattice.dim
        if manifold.dim != n:
            raise ValueError("manifold and lattice dimension mismatch")
        if not hasattr(manifold, "device_field"):
            raise TypeError("manifold has no device field; see ImplicitManifold.device_field")
        self.manifold = manifold
        self.cfg = cfg
        self.n = n
        self.ctx = _cabi.context()
        offset = np.asarray(cfg.lattice.offset, dtype=np.float64)
        lo = hi = None
        if cfg.box is not None:
            lo = np.ascontiguousarray(cfg.box[0], dtype=np.float64)
            hi = np.ascontiguousarray(cfg.box[1], dtype=np.float64)
            if lo.shape != (n,) or hi.shape != (n,) or np.any(lo >= hi):
                raise ValueError("box must be a (lower, upper) pair with lower < upper")
        h = C.c_void_p()
        _cabi.check(_cabi.lib.pt_trace_create(
            self.ctx.handle, manifold.device_field(), n, cfg.lattice.scale, offset.ctypes.data,
            lo.ctypes.data if lo is not None else None, hi.ctypes.data if hi is not None else None,
            min(int(cfg.max_edges), (1 << 31) - 2), float(cfg.eps), C.byref(h)))
        self.handle = h

    def __del__(self):
        h, self.handle = getattr(self, "handle", None), None
        if h:
            try:
                _cabi.lib.pt_trace_destroy(h)
            except Exception:
                pass

    # -- thin wrappers ----------------------------------------------------------------------
    def _seeds(self, seeds) -> np.ndarray:
        s = np.ascontiguousarray(np.atleast_2d(np.asarray(seeds, dtype=np.float64)))
        if s.shape[0] == 0 or s.shape[1] != self.n:
            raise ValueError("seeds must be a non-empty (m, n) array")
        if not np.isfinite(s).all():
            raise ValueError("point coordinates must be finite")
        return s

    def locate(self, seeds):
        s = self._seeds(seeds)
        _cabi.check(_cabi.lib.pt_trace_locate(self.handle, s.ctypes.data, s.shape[0]))

    def run(self, seeds):
        s = self._seeds(seeds)
        _cabi.check(_cabi.lib.pt_trace_run(self.handle, s.ctypes.data, s.shape[0]))

    def expand(self) -> int:
        out = C.c_longlong(0)
        _cabi.check(_cabi.lib.pt_trace_expand(self.handle, C.byref(out)))
        return int(out.value)

    def raw_stats(self) -> _cabi.TraceStats:
        st = _cabi.TraceStats()
        _cabi.check(_cabi.lib.pt_trace_get_stats(self.handle, C.byref(st)))
        return st

    def stats(self) -> TraceStats:
        st = self.raw_stats()
        rows = np.zeros((int(st.n_stages), 5), dtype=np.int64)
        if rows.shape[0]:
            _cabi.check(_cabi.lib.pt_trace_stages(self.handle, rows.ctypes.data, rows.shape[0]))
        return TraceStats(
            levels=int(st.levels), seeds=int(st.seeds), visited_edges=int(st.visited_edges),
            field_evaluations=int(st.field_evaluations), dropped_out_of_box=int(st.dropped_out_of_box),
            complete=bool(st.complete), closure_ok=bool(st.closure_ok), ambiguous_signs=int(st.ambiguous_signs),
            stages=[StageStat(_STAGE_NAMES[int(r[0])], int(r[1]), int(r[2]), int(r[3]), int(r[4])) for r in rows],
        )

    def edge_arrays(self, first=0, count=None):
        total = int(self.raw_stats().visited_edges)
        count = total - first if count is None else count
        base = np.empty((count, self.n), dtype=np.int32)
        mask = np.empty(count, dtype=np.uint32)
        sa = np.empty(count, dtype=np.int8)
        if count:
            _cabi.check(_cabi.lib.pt_trace_edges(self.handle, first, count, base.ctypes.data,
                                                 mask.ctypes.data, sa.ctypes.data))
        return base, mask, sa

    def points(self) -> np.ndarray:
        total = int(self.raw_stats().visited_edges)
        out = np.zeros((total, self.n), dtype=np.float64)
        if total:
            _cabi.check(_cabi.lib.pt_trace_points(self.handle, out.ctypes.data))
        return out

    def adjacency(self) -> np.ndarray:
        count = int(_cabi.lib.pt_trace_adjacency(self.handle, None, 0))
        if count < 0:
            _cabi.check(count)
        pairs = np.empty((count, 2), dtype=np.int64)
        if count:
            _cabi.lib.pt_trace_adjacency(self.handle, pairs.ctypes.data, count)
        return pairs


class _LazyEdges(Sequence):
    """List-like view of the traced edges; PermSimplex objects are built on first use."""

    def __init__(self, handle: _TraceHandle, count: int):
        self._handle = handle
        self._count = count
        self._arrays = None
        self._list = None

    def arrays(self):
        """(base[E, n] int32, mask[E] uint32, sign_a[E] int8) in admission order."""
        if self._arrays is None:
            self._arrays = self._handle.edge_arrays(0, self._count)
        return self._arrays

    def _materialise(self):
        if self._list is None:
            base, mask, _ = self.arrays()
            self._list = edges_from_arrays(base, mask)
        return self._list

    def __len__(self):
        return self._count

    def __bool__(self):
        return self._count > 0

    def __getitem__(self, i):
        return self._materialise()[i]

    def __iter__(self):
        return iter(self._materialise())

    def __eq__(self, other):
        return list(self) == list(other)

    def __repr__(self):
        return f"<{self._count} traced edges>"


class TraceResult:
    """Traced edges, one intersection point per edge, and coface adjacency (tracer.py:99-120).

    `edges` / `adjacency` are lazy views over device arrays; `device` is the live trace the
    refinement stage continues from without a host round trip.
    """

    def __init__(self, handle: _TraceHandle | None, stats: TraceStats, config: TraceConfig,
                 points: np.ndarray | None = None, edges=None, adjacency=None):
        self.device = handle
        self.stats = stats
        self.config = config
        self._edges = edges if edges is not None else _LazyEdges(handle, stats.visited_edges)
        self._points = points
        self._adjacency = adjacency

    @property
    def edges(self):
        return self._edges

    @property
    def points(self) -> np.ndarray:
        if self._points is None:
            self._points = self.device.points()
        return self._points

    @property
    def adjacency(self) -> list[tuple[int, int]]:
        if self._adjacency is None:
            self._adjacency = [(int(i), int(j)) for i, j in self.device.adjacency()]
        return self._adjacency

    @property
    def complete(self) -> bool:
        return self.stats.complete

    @property
    def closure_ok(self) -> bool:
        return self.stats.closure_ok


def _frontier_from_device(handle: _TraceHandle, capacity: int) -> Frontier:
    first, count = C.c_longlong(0), C.c_longlong(0)
    _cabi.check(_cabi.lib.pt_trace_frontier(handle.handle, C.byref(first), C.byref(count)))
    base, mask, sa = handle.edge_arrays(int(first.value), int(count.value))
    edges = tuple(edges_from_arrays(base, mask))
    signs = tuple((int(s), -int(s)) for s in sa)
    return Frontier(edges=edges, capacity=capacity, signs=signs)


def locate_edges(seeds, manifold, cfg: TraceConfig) -> Frontier:
    """Initial frontier: deduplicated sign-changing edges of the seed cells (tracer.py:409-415)."""
    handle = _TraceHandle(manifold, cfg)
    handle.locate(seeds)
    st = handle.stats()
    capacity = next((s.capacity for s in st.stages if s.name == "cell_edges"), 0)
    return _frontier_from_device(handle, capacity)


def expand_frontier(frontier: Frontier, visited, manifold, cfg: TraceConfig) -> Frontier:
    """One BFS level; `visited` (a set of canonical edges) gains the new edges (tracer.py:418-433)."""
    handle = _TraceHandle(manifold, cfg)
    n = cfg.lattice.dim
    seen = list(visited)
    vb, vm = edges_to_arrays(seen, n)
    fb, fm = edges_to_arrays(list(frontier.edges), n)
    base = np.ascontiguousarray(np.vstack([vb, fb]).astype(np.int32))
    mask = np.ascontiguousarray(np.concatenate([vm, fm]).astype(np.uint32))
    _cabi.check(_cabi.lib.pt_trace_seed_edges(handle.handle, base.ctypes.data, mask.ctypes.data,
                                              len(seen), len(frontier.edges)))
    handle.expand()
    st = handle.stats()
    capacity = next((s.capacity for s in st.stages if s.name == "coface_partner"), 0)
    out = _frontier_from_device(handle, capacity)
    visited.update(out.edges)
    return out


def trace(seeds, manifold, cfg: TraceConfig) -> TraceResult:
    """Breadth-first closure of sign-changing edges reachable from the seeds (tracer.py:436-452)."""
    handle = _TraceHandle(manifold, cfg)
    handle.run(seeds)
    stats = handle.stats()
    result = TraceResult(handle, stats, cfg)
    result._points = handle.points() if stats.visited_edges else np.zeros((0, cfg.lattice.dim))
    if cfg.lattice.dim == 2 and stats.visited_edges:
        degree = np.zeros(stats.visited_edges, dtype=np.int64)
        pairs = handle.adjacency()
        np.add.at(degree, pairs[:, 0], 1)
        np.add.at(degree, pairs[:, 1], 1)
        stats.polyline_closed = bool(np.all(degree == 2))
    return result


# ---- EDGEMESH v1 (tracer.py:455-488): repr() reals, exact round trip --------------------------------

def write_edgemesh(target, dim, points, pairs) -> None:
    points = np.asarray(points, dtype=np.float64)
    rows = [f"EDGEMESH n {dim} V {len(points)} E {len(pairs)}"]
    rows += [" ".join(repr(float(v)) for v in p) for p in points]
    rows += [f"{i} {j}" for i, j in pairs]
    text = "\n".join(rows) + "\n"
    if hasattr(target, "write"):
        target.write(text)
    else:
        Path(target).write_text(text)


def read_edgemesh(source):
    text = source.read() if hasattr(source, "read") else Path(source).read_text()
    lines = [ln for ln in text.splitlines() if ln.strip()]
    if not lines:
        raise ValueError("empty edgemesh")
    head = lines[0].split()
    if len(head) != 7 or (head[0], head[1], head[3], head[5]) != ("EDGEMESH", "n", "V", "E"):
        raise ValueError(f"malformed edgemesh header: {lines[0]!r}")
    dim, nv, ne = int(head[2]), int(head[4]), int(head[6])
    if len(lines) != 1 + nv + ne:
        raise ValueError("edgemesh line count does not match header")
    points = np.array([[float(v) for v in ln.split()] for ln in lines[1:1 + nv]])
    points = points.reshape(nv, dim) if nv else np.zeros((0, dim))
    pairs = [tuple(int(v) for v in ln.split()) for ln in lines[1 + nv:]]
    return dim, points, pairs
