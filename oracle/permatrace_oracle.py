"""CPU oracle: a restatement of the reference's hot-path algorithms.

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs, never by paper_2406_04795_b200 (the product path has no CPU
fallback and fails loudly without its CUDA library).

PARITY PINNED: tests/test_oracle_golden.py checks every function here against golden vectors
generated from the real reference (tests/golden/make_golden.py imports /root/reference/pkg/src with
its Cython backend): expansion plans and cell cofaces for all edge types n=2..6, ordered traces of
analytic and learned manifolds n=2..6, refinement output, FK and collision masks, and the
reference's own known-answer vectors (test_backends.py dyadic touches, test_lattice.py Fig. 2).

Representation (plain Python, nothing shared with the product):
    vertex = tuple of ints;  simplex = (base vertex, parts) with parts a tuple of sorted label tuples,
    exactly the reference's PermSimplex fields so results compare field by field.
Every function cites the reference lines it follows (paths under /root/reference/pkg/src/permatrace/).
"""

from __future__ import annotations

import ctypes
import os
from itertools import permutations, product
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB = None


def _kernels():
    """liboracle_kernels.so (oracle/kernels.c); built by `make -C oracle` / __graft_entry__.build()."""
    global _LIB
    if _LIB is None:
        path = _HERE / "liboracle_kernels.so"
        if not path.exists():
            raise ImportError(f"{path} missing: run `make -C {_HERE}`")
        lib = ctypes.CDLL(str(path))
        vp, ll, d, i = ctypes.c_void_p, ctypes.c_ssize_t, ctypes.c_double, ctypes.c_int
        lib.oracle_rbf_values.argtypes = [vp, ll, i, vp, ll, vp, d, d, vp]
        lib.oracle_rbf_values_mt.argtypes = [vp, ll, i, vp, ll, vp, d, d, vp, i]
        lib.oracle_sphere_box_hits.argtypes = [vp, vp, ll, d, d, d, vp]
        lib.oracle_sphere_cylinder_hits.argtypes = [vp, vp, ll, d, d, vp]
        lib.oracle_sphere_sphere_hits.argtypes = [vp, vp, ll, d, vp]
        for fn in (lib.oracle_rbf_values, lib.oracle_rbf_values_mt, lib.oracle_sphere_box_hits,
                   lib.oracle_sphere_cylinder_hits, lib.oracle_sphere_sphere_hits):
            fn.restype = None
        _LIB = lib
    return _LIB


THREADS = 1   # bench.py raises this for the CPU-baseline leg (rows are independent)


# =================================================================================================
# backend kernels (_kernels.pyx)
# =================================================================================================

def rbf_values(points, support, weights, gamma, bias):
    """_kernels.pyx:18-40."""
    points = np.ascontiguousarray(points, dtype=np.float64)
    support = np.ascontiguousarray(support, dtype=np.float64)
    weights = np.ascontiguousarray(weights, dtype=np.float64)
    if support.shape[1] != points.shape[1] or weights.shape[0] != support.shape[0]:
        raise ValueError("support/weights shape mismatch")
    out = np.empty(points.shape[0], dtype=np.float64)
    lib = _kernels()
    if THREADS > 1:
        lib.oracle_rbf_values_mt(points.ctypes.data, points.shape[0], points.shape[1], support.ctypes.data,
                                 support.shape[0], weights.ctypes.data, float(gamma), float(bias),
                                 out.ctypes.data, int(THREADS))
    else:
        lib.oracle_rbf_values(points.ctypes.data, points.shape[0], points.shape[1], support.ctypes.data,
                              support.shape[0], weights.ctypes.data, float(gamma), float(bias), out.ctypes.data)
    return out


def _hits(fn, centers, radii, *params):
    centers = np.ascontiguousarray(centers, dtype=np.float64)
    radii = np.ascontiguousarray(radii, dtype=np.float64)
    out = np.zeros(centers.shape[0], dtype=np.uint8)
    fn(centers.ctypes.data, radii.ctypes.data, centers.shape[0], *[float(p) for p in params], out.ctypes.data)
    return out


def sphere_box_hits(centers, radii, lx, ly, lz):
    """_kernels.pyx:43-76."""
    return _hits(_kernels().oracle_sphere_box_hits, centers, radii, lx, ly, lz)


def sphere_cylinder_hits(centers, radii, height, radius):
    """_kernels.pyx:79-104."""
    return _hits(_kernels().oracle_sphere_cylinder_hits, centers, radii, height, radius)


def sphere_sphere_hits(centers, radii, radius):
    """_kernels.pyx:107-122."""
    return _hits(_kernels().oracle_sphere_sphere_hits, centers, radii, radius)


# =================================================================================================
# lattice (lattice.py)
# =================================================================================================

def part_step(part, n):
    """lattice.py:95-107: label i<n steps +e_i, label n steps -(1..1)."""
    s = [0] * n
    for label in part:
        if label != n:
            s[label] += 1
    if n in part:
        s = [v - 1 for v in s]
    return tuple(s)


def vadd(v, d):
    return tuple(a + b for a, b in zip(v, d))


def simplex_vertices(simplex):
    """lattice.py:114-122."""
    base, parts = simplex
    n = len(base)
    verts = [tuple(base)]
    for part in parts[:-1]:
        verts.append(vadd(verts[-1], part_step(part, n)))
    return verts


def edge_vertices(edge):
    """lattice.py:125-127."""
    base, parts = edge
    return tuple(base), vadd(base, part_step(parts[0], len(base)))


def canonicalize(simplex):
    """lattice.py:156-166: rotate the cycle to the lexicographically smallest vertex."""
    base, parts = simplex
    verts = simplex_vertices(simplex)
    j = min(range(len(verts)), key=lambda i: verts[i])
    if j == 0:
        return (tuple(base), tuple(parts))
    return (verts[j], tuple(parts[j:]) + tuple(parts[:j]))


def locate_point(point, scale, offset):
    """lattice.py:135-153."""
    p = np.asarray(point, dtype=np.float64)
    n = p.size
    y = (p - np.asarray(offset)) / scale
    base = np.floor(y)
    frac = y - base
    order = sorted(range(n), key=lambda i: (-frac[i], i))
    return (tuple(int(b) for b in base), tuple((i,) for i in order) + ((n,),))


def _merged(parts):
    return tuple(sorted(x for p in parts for x in p))


def pair_edges(simplex):
    """lattice.py:182-193: canonical edge per cycle-vertex pair a<b (a outer)."""
    base, parts = simplex
    verts = simplex_vertices(simplex)
    k = len(parts) - 1
    out = []
    for a in range(k + 1):
        for b in range(a + 1, k + 1):
            out.append(canonicalize((verts[a], (_merged(parts[a:b]), _merged(parts[b:] + parts[:a])))))
    return out


def ordered_splits(part):
    """lattice.py:210-218."""
    m = len(part)
    for bits in range(1, (1 << m) - 1):
        yield (tuple(part[i] for i in range(m) if bits >> i & 1),
               tuple(part[i] for i in range(m) if not bits >> i & 1))


def cofaces2_of_edge(edge):
    """lattice.py:221-242."""
    base, (p1, p2) = edge
    out = [canonicalize((base, (s1, s2, p2))) for s1, s2 in ordered_splits(p1)]
    out += [canonicalize((base, (p1, t1, t2))) for t1, t2 in ordered_splits(p2)]
    return out


def cellcofaces_of_edge(edge):
    """lattice.py:245-266."""
    base, (p1, p2) = edge
    out, seen = [], set()
    for o1 in permutations(p1):
        for o2 in permutations(p2):
            cell = canonicalize((base, tuple((x,) for x in o1 + o2)))
            if cell not in seen:
                seen.add(cell)
                out.append(cell)
    return out


_PLAN_CACHE: dict = {}


def expansion_plan(parts, n):
    """tracer.py:123-149: per coface (third-vertex offset, partner (b,c), partner (a,c)), each
    partner as (base offset, parts, base-is-the-shared-endpoint)."""
    key = (parts, n)
    if key in _PLAN_CACHE:
        return _PLAN_CACHE[key]
    origin = (0,) * n
    edge = (origin, parts)
    a, b = edge_vertices(edge)
    plan = []
    for face in cofaces2_of_edge(edge):
        c = next(v for v in simplex_vertices(face) if v != a and v != b)
        bc = ac = None
        for e2 in pair_edges(face):
            p, q = edge_vertices(e2)
            if {p, q} == {b, c}:
                bc = (e2[0], e2[1], p == b)
            elif {p, q} == {a, c}:
                ac = (e2[0], e2[1], p == a)
        assert bc is not None and ac is not None
        plan.append((c, bc, ac))
    _PLAN_CACHE[key] = tuple(plan)
    return _PLAN_CACHE[key]


# =================================================================================================
# manifolds (manifold.py)
# =================================================================================================

class Field:
    """values/signs of one implicit manifold.

    kind "rbf": F = rbf_values(...) - barrier (manifold.py:203-208, :165-169)
    kind "sphere"/"ellipsoid"/"plane": manifold.py:85-87, :110-112, :133-134
    """

    def __init__(self, kind, dim, **kw):
        self.kind, self.dim = kind, dim
        self.__dict__.update(kw)
        self.evaluations = 0

    @classmethod
    def rbf(cls, support, weights, gamma, bias=0.0, barrier=None):
        support = np.ascontiguousarray(support, dtype=np.float64)
        return cls("rbf", support.shape[1], support=support,
                   weights=np.ascontiguousarray(weights, dtype=np.float64), gamma=float(gamma),
                   bias=float(bias), barrier=barrier)

    @classmethod
    def sphere(cls, center, radius):
        center = np.asarray(center, dtype=np.float64)
        return cls("sphere", center.size, center=center, radius=float(radius))

    @classmethod
    def ellipsoid(cls, center, semi_axes):
        center = np.asarray(center, dtype=np.float64)
        return cls("ellipsoid", center.size, center=center, semi_axes=np.asarray(semi_axes, dtype=np.float64))

    @classmethod
    def plane(cls, normal, offset):
        normal = np.asarray(normal, dtype=np.float64)
        return cls("plane", normal.size, normal=normal, offset=float(offset))

    def values(self, points):
        pts = np.ascontiguousarray(points, dtype=np.float64)
        self.evaluations += pts.shape[0]
        if self.kind == "rbf":
            out = rbf_values(pts, self.support, self.weights, self.gamma, self.bias)
            if self.barrier is not None:
                scale, gain, lower, upper = self.barrier
                low = np.logaddexp(0.0, (np.asarray(lower) - pts) / scale)
                high = np.logaddexp(0.0, (pts - np.asarray(upper)) / scale)
                out -= gain * scale * (low + high).sum(axis=1)
            return out
        if self.kind == "sphere":
            d = pts - self.center
            return np.einsum("ij,ij->i", d, d) - self.radius ** 2
        if self.kind == "ellipsoid":
            d = (pts - self.center) / self.semi_axes
            return np.einsum("ij,ij->i", d, d) - 1.0
        return pts @ self.normal - self.offset

    def signs(self, points):
        """manifold.py:71-72: +1 where F > 0 else -1."""
        return np.where(self.values(points) > 0.0, 1, -1).astype(np.int8)


def intersection_points_batch(field, a, b, eps, signs_a=None):
    """manifold.py:351-383: per-row bisection until seg*(hi-lo) <= eps."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape[0] == 0:
        return a.copy()
    if signs_a is None:
        signs_a = field.signs(a)
    signs_a = np.asarray(signs_a)
    seg = np.linalg.norm(b - a, axis=1)
    lo = np.zeros(a.shape[0])
    hi = np.ones(a.shape[0])
    diff = b - a
    active = np.nonzero(seg > eps)[0]
    while active.size:
        mid = 0.5 * (lo[active] + hi[active])
        s = field.signs(a[active] + mid[:, None] * diff[active])
        same = s == signs_a[active]
        lo[active] = np.where(same, mid, lo[active])
        hi[active] = np.where(same, hi[active], mid)
        active = active[seg[active] * (hi[active] - lo[active]) > eps]
    t = 0.5 * (lo + hi)
    return a + t[:, None] * diff


# =================================================================================================
# tracer (tracer.py)
# =================================================================================================

class Trace:
    """Restatement of _Tracer (tracer.py:152-406) with plain dict/set bookkeeping."""

    def __init__(self, field, n, scale, offset=None, box=None, max_edges=10_000_000, eps=1e-9):
        self.f, self.n, self.scale = field, n, float(scale)
        self.offset = np.zeros(n) if offset is None else np.asarray(offset, dtype=np.float64)
        self.max_edges, self.eps = max_edges, eps
        self.sign_of: dict = {}
        self.visited: dict = {}
        self.edge_signs: list = []
        self.adjacency: set = set()
        self.levels = self.seeds = self.field_evaluations = self.dropped = 0
        self.candidates = 0
        self.complete = True
        self.stages: list = []
        if box is not None:
            self.lo = (np.asarray(box[0], dtype=np.float64) - self.offset) / self.scale   # tracer.py:174-175
            self.hi = (np.asarray(box[1], dtype=np.float64) - self.offset) / self.scale
        else:
            self.lo = self.hi = None

    def in_box(self, v):
        """tracer.py:187-193."""
        if self.lo is None:
            return True
        return all(self.lo[i] <= c <= self.hi[i] for i, c in enumerate(v))

    def ensure_signs(self, vertices):
        """tracer.py:195-209."""
        unknown, local = [], set()
        for v in vertices:
            if v not in self.sign_of and v not in local:
                local.add(v)
                unknown.append(v)
        if not unknown:
            return
        pts = np.asarray(unknown, dtype=np.float64) * self.scale + self.offset
        vals = self.f.values(pts)
        self.field_evaluations += len(unknown)
        for v, val in zip(unknown, vals):
            self.sign_of[v] = 1 if val > 0.0 else -1

    def admit(self, edge, s_pair, source=None):
        """tracer.py:239-252."""
        idx = self.visited.get(edge)
        if idx is None:
            if len(self.visited) >= self.max_edges:
                self.complete = False
                return None
            idx = len(self.visited)
            self.visited[edge] = idx
            self.edge_signs.append(s_pair)
        if source is not None and source != idx:
            self.adjacency.add((source, idx) if source < idx else (idx, source))
        return idx

    def locate(self, seeds):
        """tracer.py:256-301; returns the list of (edge, sign pair) frontier entries."""
        seeds = np.atleast_2d(np.asarray(seeds, dtype=np.float64))
        self.seeds += seeds.shape[0]
        cells = [locate_point(s, self.scale, self.offset) for s in seeds]
        self.stages.append(("locate_cells", self.levels, len(cells), len(cells), len(cells)))
        verts = [v for c in cells for v in simplex_vertices(c)]
        self.ensure_signs(verts)
        entries, batch, produced = [], set(), 0
        for cell in cells:
            for edge in pair_edges(cell):
                va, vb = edge_vertices(edge)
                sa, sb = self.sign_of[va], self.sign_of[vb]
                if sa == sb:
                    continue
                produced += 1
                if not (self.in_box(va) and self.in_box(vb)):
                    self.dropped += 1
                    continue
                if edge in batch or edge in self.visited:
                    continue
                batch.add(edge)
                entries.append((edge, (sa, sb)))
        bound = (self.n + 1) * self.n // 2
        self.stages.append(("cell_edges", self.levels, len(cells), len(cells) * bound, produced))
        return entries

    def expand(self, entries):
        """tracer.py:322-380."""
        self.levels += 1
        n = self.n
        records = []
        for edge, s_pair in entries:
            for plan_entry in expansion_plan(edge[1], n):
                records.append((edge, s_pair, plan_entry))
        self.candidates += len(records)
        self.stages.append(("edge_cofaces", self.levels, len(entries), len(records), len(records)))
        self.ensure_signs([vadd(r[0][0], r[2][0]) for r in records])
        out, batch = [], set()
        for edge, (sa, sb), (c_off, bc, ac) in records:
            base = edge[0]
            sc = self.sign_of[vadd(base, c_off)]
            tpl, s_shared = (bc, sb) if sc == sa else (ac, sa)
            off, parts, base_is_shared = tpl
            s_pair = (s_shared, sc) if base_is_shared else (sc, s_shared)
            new_edge = (vadd(base, off), parts)
            va, vb = edge_vertices(new_edge)
            if not (self.in_box(va) and self.in_box(vb)):
                self.dropped += 1
                continue
            source = self.visited[edge]
            if new_edge in self.visited or new_edge in batch:
                self.admit(new_edge, None, source)
                continue
            idx = self.admit(new_edge, s_pair, source)
            if idx is None:
                continue
            batch.add(new_edge)
            out.append((new_edge, s_pair))
        self.stages.append(("coface_partner", self.levels, len(records), len(records), len(records)))
        return out

    def run(self, seeds):
        """tracer.py:436-452."""
        frontier = self.locate(seeds)
        for edge, s_pair in frontier:
            self.admit(edge, s_pair)
        while frontier and self.complete:
            frontier = self.expand(frontier)
        return self

    # -- result (tracer.py:384-406) --
    @property
    def edges(self):
        return list(self.visited)

    def points(self):
        edges = self.edges
        if not edges:
            return np.zeros((0, self.n))
        ends = [edge_vertices(e) for e in edges]
        a = np.asarray([p[0] for p in ends], dtype=np.float64) * self.scale + self.offset
        b = np.asarray([p[1] for p in ends], dtype=np.float64) * self.scale + self.offset
        signs_a = np.asarray([s[0] for s in self.edge_signs], dtype=np.int8)
        return intersection_points_batch(self.f, a, b, self.eps, signs_a=signs_a)

    @property
    def closure_ok(self):
        return bool(self.visited) and self.complete and self.dropped == 0

    def sorted_adjacency(self):
        return sorted(self.adjacency)


# =================================================================================================
# subdivision (subdivision.py)
# =================================================================================================

def containment_check(vertex, k):
    """subdivision.py:51-58."""
    prev = int(k)
    for c in vertex:
        if c > prev:
            return False
        prev = c
    return prev >= 0


def barycentric_weights(vertex, k):
    """subdivision.py:61-68."""
    v = np.asarray(vertex, dtype=np.float64)
    w = np.empty(v.size + 1)
    w[0] = 1.0 - v[0] / k
    w[1:-1] = (v[:-1] - v[1:]) / k
    w[-1] = v[-1] / k
    return w


def build_template(n, k):
    """subdivision.py:87-120 via the enumeration the reference's acceptance test 05 equates it to
    (pkg/tests/oracles.py:109-122): vertices passing containment_check, edges x -> x + {0,1}^n."""
    verts = sorted(v for v in product(range(k + 1), repeat=n) if containment_check(v, k))
    index = {v: i for i, v in enumerate(verts)}
    pairs = []
    for v in verts:
        for s in product((0, 1), repeat=n):
            if any(s):
                w = vadd(v, s)
                if w in index:
                    pairs.append((index[v], index[w]))
    pairs.sort()
    vertices = np.asarray(verts, dtype=np.int64)
    edges = np.asarray(pairs, dtype=np.int64).reshape(len(pairs), 2)
    weights = np.vstack([barycentric_weights(v, k) for v in verts])
    return vertices, edges, weights


def coarse_cells(edges):
    """subdivision.py:132-141."""
    out = {cell for edge in edges for cell in cellcofaces_of_edge(edge)}
    return sorted(out, key=lambda c: (c[0], c[1]))


class PointRegistry:
    """subdivision.py:195-217: eps-grid buckets, 3^n neighbourhood, first keeper wins."""

    def __init__(self, eps, n):
        self.eps = eps
        self.cells: dict = {}
        self.points: list = []
        self.neighborhood = list(product((-1, 0, 1), repeat=n))

    def add(self, p):
        key = tuple(int(c) for c in np.floor(p / self.eps))
        for off in self.neighborhood:
            bucket = self.cells.get(tuple(k + o for k, o in zip(key, off)))
            if not bucket:
                continue
            for idx in bucket:
                if float(np.linalg.norm(self.points[idx] - p)) <= self.eps:
                    return None
        idx = len(self.points)
        self.points.append(p)
        self.cells.setdefault(key, []).append(idx)
        return idx


def crossing_points(batch, template, field, scale, offset, eps):
    """subdivision.py:256-272 for one batch of cells: the bisected point of every sign-changing
    template edge, cell-major then template-edge-major (duplicates across cells included)."""
    vertices, tedges, weights = template
    n = vertices.shape[1]
    if not len(batch):
        return np.zeros((0, n))
    corners = np.asarray([simplex_vertices(c) for c in batch], dtype=np.float64)
    corners = corners * scale + np.asarray(offset, dtype=np.float64)
    fine = np.einsum("vc,bcn->bvn", weights, corners)
    signs = field.signs(fine.reshape(-1, n)).reshape(len(batch), -1)
    sa = signs[:, tedges[:, 0]]
    sb = signs[:, tedges[:, 1]]
    idx_b, idx_e = np.nonzero(sa != sb)
    if not idx_b.size:
        return np.zeros((0, n))
    a = fine[idx_b, tedges[idx_e, 0]]
    b = fine[idx_b, tedges[idx_e, 1]]
    return intersection_points_batch(field, a, b, eps, signs_a=sa[idx_b, idx_e])


def refine(cells, template, field, checker, scale, offset, k, eps, eps_dedup=None, batch_cells=None):
    """subdivision.py:220-301.  `template` = (vertices, edges, weights); returns a dict with points,
    in_collision, crossing_edges per batch, new_points per batch."""
    n = template[0].shape[1]
    cells = list(cells)
    if eps_dedup is None:
        eps_dedup = scale / (10.0 * k * k)
    step = len(cells) if not batch_cells else batch_cells
    batches = [cells[i:i + step] for i in range(0, len(cells), max(step, 1))] if cells else []
    registry = PointRegistry(eps_dedup, n)
    labels, crossing_counts, new_counts = [], [], []
    for batch in batches:
        pts = crossing_points(batch, template, field, scale, offset, eps)
        fresh = [p for p in pts if registry.add(p) is not None]
        if fresh:
            labels.extend(bool(h) for h in np.asarray(checker(np.asarray(fresh)), dtype=bool))
        crossing_counts.append(int(pts.shape[0]))
        new_counts.append(len(fresh))
    points = np.asarray(registry.points, dtype=np.float64) if registry.points else np.zeros((0, n))
    return {
        "points": points,
        "in_collision": np.asarray(labels, dtype=bool),
        "crossing_edges": crossing_counts,
        "new_points": new_counts,
        "eps_dedup": eps_dedup,
    }


# =================================================================================================
# collision (collision.py, pipeline.py:256-270)
# =================================================================================================

def axis_rotations(axis, angles):
    """collision.py:191-201 (Rodrigues)."""
    kx, ky, kz = axis
    k = np.asarray(axis, dtype=np.float64)
    skew = np.array([[0.0, -kz, ky], [kz, 0.0, -kx], [-ky, kx, 0.0]])
    c = np.cos(angles)
    s = np.sin(angles)
    return c[:, None, None] * np.eye(3) + s[:, None, None] * skew + (1.0 - c)[:, None, None] * np.outer(k, k)


def fk_batch(robot, configs):
    """collision.py:204-225.  robot = dict(joints=[dict(kind, axis, rot, trans, limits)],
    spheres=[dict(link, offset, radius)])."""
    q = np.atleast_2d(np.asarray(configs, dtype=np.float64))
    m = q.shape[0]
    rot = np.broadcast_to(np.eye(3), (m, 3, 3)).copy()
    trans = np.zeros((m, 3))
    frames = [(rot, trans)]
    for j, joint in enumerate(robot["joints"]):
        trans = np.einsum("mij,j->mi", rot, np.asarray(joint["trans"], dtype=np.float64)) + trans
        rot = np.einsum("mij,jk->mik", rot, np.asarray(joint["rot"], dtype=np.float64))
        if joint["kind"] == "revolute":
            rot = np.einsum("mij,mjk->mik", rot, axis_rotations(joint["axis"], q[:, j]))
        else:
            trans = trans + np.einsum("mij,j->mi", rot, np.asarray(joint["axis"])) * q[:, j, None]
        frames.append((rot, trans))
    centers = np.empty((m, len(robot["spheres"]), 3))
    for si, sp in enumerate(robot["spheres"]):
        frot, ftrans = frames[sp["link"]]
        centers[:, si] = np.einsum("mij,j->mi", frot, np.asarray(sp["offset"], dtype=np.float64)) + ftrans
    return centers


def obstacle_hits(centers, radii, obs):
    """collision.py:243-250; obs = dict(type, rot, trans, dims)."""
    local = np.ascontiguousarray((centers - np.asarray(obs["trans"])) @ np.asarray(obs["rot"]))   # Pose.to_local :83-84
    radii = np.ascontiguousarray(radii)
    if obs["type"] == "box":
        return sphere_box_hits(local, radii, *obs["dims"][:3])
    if obs["type"] == "cylinder":
        return sphere_cylinder_hits(local, radii, obs["dims"][0], obs["dims"][1])
    return sphere_sphere_hits(local, radii, obs["dims"][0])


def batch_hits(robot, scene, q):
    """collision.py:278-286."""
    m = q.shape[0]
    centers = fk_batch(robot, q).reshape(m * len(robot["spheres"]), 3)
    radii = np.tile(np.array([sp["radius"] for sp in robot["spheres"]]), m)
    hit = np.zeros(m, dtype=bool)
    for obs in scene:
        hit |= obstacle_hits(centers, radii, obs).reshape(m, -1).astype(bool).any(axis=1)
    return hit


def not_free(robot, scene, points, batch_size=4096):
    """pipeline.py:256-270 + batch_check(on_limit semantics of collision.py:319-329)."""
    points = np.atleast_2d(np.asarray(points, dtype=np.float64))
    lo = np.array([j["limits"][0] for j in robot["joints"]])
    hi = np.array([j["limits"][1] for j in robot["joints"]])
    out = np.ones(points.shape[0], dtype=bool)
    inside = np.all((points >= lo) & (points <= hi), axis=1)
    idx = np.nonzero(inside)[0]
    for s in range(0, idx.size, batch_size):
        chunk = idx[s:s + batch_size]
        out[chunk] = batch_hits(robot, scene, points[chunk])
    return out
