"""Symmetric k-fold subdivision of traced cells, refined in one device pass.

Public names follow ``permatrace/subdivision.py:26-40``.  `coarse_cells` and `refine` run in
``csrc/pt_cells.cu`` / ``csrc/pt_refine.cu``; the subdivision template is tiny and built on the
host by direct enumeration of the integer points of the k-scaled reference cell.

What the device path keeps from the reference, exactly:
  * cells sorted by (base, permutation)                                  subdivision.py:141
  * crossing enumeration cell-major, template-edge-major                 subdivision.py:263-266
  * bisection per crossing fine edge to `cfg.eps`                        subdivision.py:267-272
  * greedy first-keeper dedup at eps_dedup in that order                 subdivision.py:195-217, :275-278
  * results independent of the memory budget (only BatchStat rows change) subdivision.py:229-236
What it does differently: a fine vertex / fine edge shared by several coarse cells is evaluated /
root-solved once (integer fine-lattice keys), not once per cell.
"""

from __future__ import annotations

import ctypes as C
import time
from collections.abc import Sequence
from dataclasses import dataclass
from itertools import product

import numpy as np

from . import _cabi
from . import lattice
from .lattice import PermSimplex
from .tracer import TraceConfig, TraceResult

__all__ = [
    "SubdivisionTemplate", "BatchPlan", "BatchStat", "RefinedResult", "BudgetError", "RefineError",
    "containment_check", "barycentric_weights", "build_template", "local_to_global", "coarse_cells",
    "plan_batches", "refine",
]


class BudgetError(ValueError):
    """A single cell's working set exceeds the memory budget."""


class RefineError(RuntimeError):
    """The collision checker failed inside refine."""


def containment_check(vertex, k: int) -> bool:
    """k >= v_0 >= v_1 >= ... >= v_{n-1} >= 0 (membership in the k-scaled reference cell)."""
    bound = int(k)
    for c in vertex:
        if c > bound:
            return False
        bound = c
    return bound >= 0


def barycentric_weights(vertex, k: int) -> np.ndarray:
    """(1 - v_0/k, (v_0-v_1)/k, ..., (v_{n-2}-v_{n-1})/k, v_{n-1}/k)."""
    v = np.asarray(vertex, dtype=np.float64)
    w = np.empty(v.size + 1)
    w[0] = 1.0 - v[0] / k
    w[1:-1] = (v[:-1] - v[1:]) / k
    w[-1] = v[-1] / k
    return w


@dataclass(frozen=True, eq=False)
class SubdivisionTemplate:
    """Fine vertices (V, n) lex-sorted, edges (E, 2) index pairs i<j sorted, weights (V, n+1)."""

    n: int
    k: int
    vertices: np.ndarray
    edges: np.ndarray
    weights: np.ndarray


def build_template(n: int, k: int) -> SubdivisionTemplate:
    """Fine lattice restricted to the k-scaled reference cell.

    The reference flood-fills from one edge (subdivision.py:87-120); its own acceptance test 05
    shows the result equals direct enumeration: vertices are the integer points passing
    `containment_check`, edges join x and x + s for every non-zero 0/1 vector s with both ends
    inside.  Enumerated directly here.
    """
    if n < 2:
        raise ValueError("template dimension must be >= 2")
    if k < 1:
        raise ValueError("subdivision factor must be >= 1")

    def descend(prefix, bound):
        if len(prefix) == n:
            yield tuple(prefix)
            return
        for c in range(0, bound + 1):
            yield from descend(prefix + [c], c)

    verts = sorted(descend([], k))
    index = {v: i for i, v in enumerate(verts)}
    steps = [s for s in product((0, 1), repeat=n) if any(s)]
    pairs = []
    for v in verts:
        i = index[v]
        for s in steps:
            j = index.get(tuple(a + b for a, b in zip(v, s)))
            if j is not None:
                pairs.append((i, j))
    pairs.sort()
    vertices = np.asarray(verts, dtype=np.int64).reshape(len(verts), n)
    edges = np.asarray(pairs, dtype=np.int64).reshape(len(pairs), 2)
    weights = np.vstack([barycentric_weights(v, k) for v in verts])
    return SubdivisionTemplate(n=n, k=k, vertices=vertices, edges=edges, weights=weights)


def local_to_global(vertex, k: int, cell: PermSimplex, config: lattice.LatticeConfig) -> np.ndarray:
    """Map a template vertex into a coarse cell by barycentric combination."""
    if not containment_check(vertex, k):
        raise ValueError(f"vertex {tuple(vertex)} is outside the k={k} template region")
    corners = np.asarray(lattice.simplex_vertices(cell), dtype=np.float64)
    corners = corners * config.scale + np.asarray(config.offset)
    return barycentric_weights(vertex, k) @ corners


class _CellsHandle:
    def __init__(self, handle, n):
        self.handle = handle
        self.n = n

    def __del__(self):
        h, self.handle = self.handle, None
        if h:
            try:
                _cabi.lib.pt_cells_destroy(h)
            except Exception:
                pass


class CellList(Sequence):
    """Sorted coarse cells living on the device; PermSimplex objects are built on first use."""

    def __init__(self, handle: _CellsHandle):
        self.device = handle
        self._count = int(_cabi.lib.pt_cells_count(handle.handle))
        self._arrays = None
        self._list = None

    def arrays(self):
        """(base[C, n] int32, perm[C, n] uint8) in sorted order."""
        if self._arrays is None:
            n = self.device.n
            base = np.empty((self._count, n), dtype=np.int32)
            perm = np.empty((self._count, n), dtype=np.uint8)
            if self._count:
                _cabi.check(_cabi.lib.pt_cells_get(self.device.handle, 0, self._count,
                                                   base.ctypes.data, perm.ctypes.data))
            self._arrays = (base, perm)
        return self._arrays

    def _materialise(self):
        if self._list is None:
            self._list = lattice.cells_from_arrays(*self.arrays())
        return self._list

    def __len__(self):
        return self._count

    def __getitem__(self, i):
        return self._materialise()[i]

    def __iter__(self):
        return iter(self._materialise())

    def __eq__(self, other):
        return list(self) == list(other)

    def __repr__(self):
        return f"<{self._count} coarse cells>"


def coarse_cells(result: TraceResult) -> CellList:
    """Every full-dimensional cell containing a traced edge, deduplicated, sorted by
    (base, permutation) (reference subdivision.py:132-141)."""
    h = C.c_void_p()
    device = getattr(result, "device", None)
    if device is not None:
        _cabi.check(_cabi.lib.pt_cells_from_trace(device.handle, C.byref(h)))
        return CellList(_CellsHandle(h, device.n))
    edges = list(result.edges)
    n = result.config.lattice.dim
    base, mask = lattice.edges_to_arrays(edges, n)
    ctx = _cabi.context()
    _cabi.check(_cabi.lib.pt_cells_from_edges(ctx.handle, n, base.ctypes.data, mask.ctypes.data,
                                              len(edges), C.byref(h)))
    return CellList(_CellsHandle(h, n))


@dataclass(frozen=True)
class BatchPlan:
    batches: tuple[tuple[PermSimplex, ...], ...]
    bytes_per_cell: int
    memory_budget: int


def _cell_bytes(template: SubdivisionTemplate) -> int:
    """Reference accounting of one cell's working set (subdivision.py:151-156)."""
    v, n = template.vertices.shape
    e = template.edges.shape[0]
    return 8 * (v * (n + 1) + e * (2 * n + 2))


def _batch_bounds(count: int, template: SubdivisionTemplate, memory_budget: int | None):
    per_cell = _cell_bytes(template)
    if memory_budget is None:
        return ([0, count] if count else [0]), per_cell
    if per_cell > memory_budget:
        raise BudgetError(f"one cell needs {per_cell} bytes but the budget is {memory_budget}")
    step = max(1, memory_budget // per_cell)
    bounds = list(range(0, count, step)) + [count]
    return bounds, per_cell


def plan_batches(cells, template: SubdivisionTemplate, memory_budget: int) -> BatchPlan:
    """Greedy order-preserving batches under the byte budget."""
    cells = list(cells)
    bounds, per_cell = _batch_bounds(len(cells), template, memory_budget)
    batches = tuple(tuple(cells[a:b]) for a, b in zip(bounds[:-1], bounds[1:]))
    return BatchPlan(batches=batches, bytes_per_cell=per_cell, memory_budget=memory_budget)


@dataclass
class BatchStat:
    index: int
    cells: int
    fine_vertices: int
    crossing_edges: int
    new_points: int
    check_seconds: float


class RefinedResult:
    """Deduplicated fine intersection points with in-collision labels (reference
    subdivision.py:184-192).  `free_points` is materialised on first access."""

    def __init__(self, points, in_collision, free_points=None, eps_dedup=0.0, batch_stats=None, device_stats=None):
        self.points = points
        self.in_collision = in_collision
        self._free_points = free_points
        self.eps_dedup = eps_dedup
        self.batch_stats = batch_stats if batch_stats is not None else []
        self.device_stats = device_stats

    @property
    def free_points(self) -> np.ndarray:
        if self._free_points is None:
            self._free_points = self.points[~self.in_collision] if self.points.size else self.points.copy()
        return self._free_points

    def __repr__(self):
        return (f"RefinedResult(points={self.points.shape}, in_collision={int(self.in_collision.sum())}, "
                f"eps_dedup={self.eps_dedup!r}, batches={len(self.batch_stats)})")


class _RefineHandle:
    def __init__(self, handle):
        self.handle = handle

    def __del__(self):
        h, self.handle = self.handle, None
        if h:
            try:
                _cabi.lib.pt_refine_destroy(h)
            except Exception:
                pass


def refine(cells, template: SubdivisionTemplate, manifold, checker, cfg: TraceConfig,
           memory_budget: int | None = None, eps_dedup: float | None = None) -> RefinedResult:
    """Subdivide the cells, bisect sign-changing fine edges, dedup and label the points
    (reference subdivision.py:220-301).

    `checker` is either the device checker returned by ``pipeline._not_free_checker`` (labels are
    computed by ``pt_check_kernel`` without leaving the GPU) or any callable
    ``(m, n) float64 -> bool[m]``, which is then invoked once per batch on the host with that
    batch's fresh points, exactly like the reference (exceptions -> RefineError).
    """
    n = template.n
    if cfg.lattice.dim != n:
        raise ValueError("template and lattice dimension mismatch")
    if eps_dedup is None:
        eps_dedup = cfg.lattice.scale / (10.0 * template.k * template.k)
    if eps_dedup <= 0:
        raise ValueError("eps_dedup must be positive")
    if not hasattr(manifold, "device_field"):
        raise TypeError("manifold has no device field; see ImplicitManifold.device_field")
    ctx = _cabi.context()
    if isinstance(cells, CellList):
        cell_handle = cells.device
        count = len(cells)
    else:
        cells = list(cells)
        count = len(cells)
        base, perm = lattice.cells_to_arrays(cells, n)
        h = C.c_void_p()
        _cabi.check(_cabi.lib.pt_cells_from_host(ctx.handle, n, base.ctypes.data, perm.ctypes.data,
                                                 count, C.byref(h)))
        cell_handle = _CellsHandle(h, n)
    bounds, _ = _batch_bounds(count, template, memory_budget)
    nb = len(bounds) - 1
    bounds_arr = np.asarray(bounds, dtype=np.int64)
    tv = np.ascontiguousarray(template.vertices, dtype=np.int32)
    te = np.ascontiguousarray(template.edges, dtype=np.int32)
    offset = np.asarray(cfg.lattice.offset, dtype=np.float64)
    device_checker = getattr(checker, "device_checker", None)
    out = C.c_void_p()
    _cabi.check(_cabi.lib.pt_refine_run(
        ctx.handle, manifold.device_field(), cell_handle.handle, n, cfg.lattice.scale, offset.ctypes.data,
        template.k, tv.shape[0], tv.ctypes.data, te.shape[0], te.ctypes.data, float(cfg.eps),
        float(eps_dedup), device_checker.handle if device_checker is not None else None,
        bounds_arr.ctypes.data, nb, C.byref(out)))
    res = _RefineHandle(out)
    st = _cabi.RefineStats()
    _cabi.check(_cabi.lib.pt_refine_get_stats(res.handle, C.byref(st)))
    total = int(st.points)
    # large results land in page-locked memory: the device->host copy runs at PCIe speed without staging
    points = _cabi.pinned_empty((total, n), np.float64, ctx)
    labels = _cabi.pinned_empty((total,), np.uint8, ctx)
    if total:
        _cabi.check(_cabi.lib.pt_refine_points(res.handle, points.ctypes.data, labels.ctypes.data, None))
    rows = np.zeros((max(nb, 1), 2), dtype=np.int64)
    if nb:
        _cabi.check(_cabi.lib.pt_refine_batch_stats(res.handle, rows.ctypes.data, nb))
    seconds = [0.0] * nb
    if device_checker is None and checker is not None:
        # arbitrary host callable: one call per batch with that batch's fresh points
        labels = np.zeros(total, dtype=bool)
        at = 0
        for bi in range(nb):
            fresh = int(rows[bi, 1])
            if fresh:
                chunk = points[at:at + fresh]
                t0 = time.perf_counter()
                try:
                    hit = np.asarray(checker(chunk), dtype=bool)
                except Exception as exc:
                    raise RefineError(f"collision checker failed in batch {bi}: {exc}") from exc
                seconds[bi] = time.perf_counter() - t0
                if hit.shape != (fresh,):
                    raise RefineError(f"checker returned shape {hit.shape} in batch {bi}")
                labels[at:at + fresh] = hit
            at += fresh
    in_collision = labels.view(np.bool_) if labels.dtype == np.uint8 else labels.astype(bool)
    stats = [
        BatchStat(bi, bounds[bi + 1] - bounds[bi], (bounds[bi + 1] - bounds[bi]) * tv.shape[0],
                  int(rows[bi, 0]), int(rows[bi, 1]), seconds[bi])
        for bi in range(nb)
    ]
    device_stats = {name: int(getattr(st, name)) for name, _ in _cabi.RefineStats._fields_}
    return RefinedResult(points, in_collision, None, float(eps_dedup), stats, device_stats)
