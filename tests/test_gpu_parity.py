"""GPU parity tests: the CUDA path (through the C ABI) against the reference's golden vectors and
the CPU oracle on the same seeded inputs.  Bit-exact for integer / index / boolean results;
intersection points within 1e-5 relative (BASELINE.json north_star) -- in practice ~1e-12."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2406_04795_b200 as P
from paper_2406_04795_b200 import backend as B, collision as CO, lattice as L, manifold as M, subdivision as S, tracer as T
from oracle import permatrace_oracle as O
from tests.conftest import (ANALYTIC_TRACES, LEARNED_TRACES, PRISM_ROBOT, PRISM_SCENE, analytic_spec, oracle_model,
                            robot_scene_dicts, trace_inputs)

import os
from paper_2406_04795_b200 import _cabi


@pytest.fixture(autouse=True, params=["fp64", "fast"])
def precision_mode(request, monkeypatch):
    """Every parity test runs twice: plain fp64 bisection and the fp32-screened / Newton fast path.
    Both must return the reference's dyadic bracket midpoints."""
    monkeypatch.setenv("PERMATRACE_B200_PRECISION", "1" if request.param == "fast" else "0")
    return request.param


POINT_RTOL = 1e-5     # north_star tolerance for intersection points
POINT_ATOL = 1e-8     # what we actually hold (bracket is 1e-9)


def product_manifold(g, tag):
    if tag.startswith("kclf"):
        gbb, bar = g[f"{tag}_gbb"], g[f"{tag}_barrier"]
        n = g[f"{tag}_support"].shape[1]
        barrier = M.BoxBarrier(bar[2:2 + n], bar[2 + n:], bar[0], bar[1])
        return M.KernelClassifierManifold(g[f"{tag}_support"], g[f"{tag}_weights"], gbb[0], gbb[1], barrier=barrier)
    kind, args = analytic_spec(tag)
    return {"sphere": M.SphereManifold, "ellipsoid": M.EllipsoidManifold, "plane": M.PlaneManifold}[kind](*args)


def oracle_field(g, tag):
    from tests.test_oracle_golden import oracle_field as f
    return f(g, tag)


def product_cfg(inp):
    return T.TraceConfig(L.LatticeConfig(inp["n"], inp["scale"], inp["offset"]), box=inp["box"],
                         max_edges=inp["max_edges"], eps=inp["eps"])


# ---- B1 seam ---------------------------------------------------------------------------------------
def test_backend_seam(golden):
    g = golden("backend")
    gamma, bias = g["rbf_params"]
    got = B.rbf_values(g["rbf_points"], g["rbf_support"], g["rbf_weights"], gamma, bias)
    tol = 1e-12 * (np.abs(g["rbf_weights"]).sum() + abs(bias))          # pkg/tests/test_backends.py:90-93
    assert got.dtype == np.float64 and np.max(np.abs(got - g["rbf_values"])) <= tol
    c, r = g["hits_centers"], g["hits_radii"]
    assert np.array_equal(B.sphere_box_hits(c, r, 0.8, 0.5, 1.1), g["hits_box"])
    assert np.array_equal(B.sphere_cylinder_hits(c, r, 0.9, 0.4), g["hits_cyl"])
    assert np.array_equal(B.sphere_sphere_hits(c, r, 0.6), g["hits_sph"])
    tc, tr = g["touch_centers"], g["touch_radii"]
    assert list(B.sphere_box_hits(tc, tr, 2.0, 2.0, 2.0)) == [1, 0, 0, 1, 0]
    assert np.array_equal(B.sphere_cylinder_hits(tc, tr, 2.0, 1.0), g["touch_cyl"])
    assert np.array_equal(B.sphere_sphere_hits(tc, tr, 1.0), g["touch_sph"])
    assert B.sphere_box_hits(c, r, 0.8, 0.5, 1.1).dtype == np.uint8


def test_backend_edge_cases():
    pts = np.random.default_rng(0).normal(size=(7, 3))
    assert np.array_equal(B.rbf_values(pts, np.zeros((0, 3)), np.zeros(0), 1.0, 0.75), np.full(7, 0.75))   # bias only
    assert B.rbf_values(np.zeros((0, 3)), np.zeros((4, 3)), np.ones(4), 1.0, 0.0).shape == (0,)
    assert B.sphere_sphere_hits(np.zeros((0, 3)), np.zeros(0), 1.0).shape == (0,)
    with pytest.raises(ValueError, match="shape mismatch"):
        B.rbf_values(pts, np.zeros((4, 2)), np.ones(4), 1.0, 0.0)
    with pytest.raises(ValueError, match="shape mismatch"):
        B.rbf_values(pts, np.zeros((4, 3)), np.ones(5), 1.0, 0.0)
    # large batch, every lane-group configuration (G = 32, 4, 1) must agree
    rng = np.random.default_rng(1)
    sup, w = rng.normal(size=(700, 5)), rng.normal(size=700)
    big = rng.normal(size=(400000, 5))
    full = B.rbf_values(big, sup, w, 0.5, 0.1)
    tol = 1e-12 * (np.abs(w).sum() + 0.1)
    assert np.max(np.abs(full[:50] - B.rbf_values(big[:50], sup, w, 0.5, 0.1))) <= tol
    assert np.max(np.abs(full[:100000] - B.rbf_values(big[:100000], sup, w, 0.5, 0.1))) <= tol
    assert np.max(np.abs(full[:3000] - O.rbf_values(big[:3000], sup, w, 0.5, 0.1))) <= tol


# ---- fields ------------------------------------------------------------------------------------------
@pytest.mark.parametrize("tag", LEARNED_TRACES)
def test_learned_field_values_and_signs(golden, tag):
    g = golden("traces")
    m = product_manifold(g, tag)
    pts, want = g[f"{tag}_probe_points"], g[f"{tag}_probe_values"]
    got = m.values(pts)
    tol = 1e-12 * (np.abs(m.weights).sum() + abs(m.bias)) + 1e-13 * np.abs(want)
    assert np.all(np.abs(got - want) <= tol)
    clear = np.abs(want) > 10 * tol
    assert np.array_equal(m.signs(pts)[clear], np.where(want > 0, 1, -1)[clear])
    assert m.signs(pts).dtype == np.int8
    assert abs(m.value(pts[0]) - want[0]) <= tol[0]


@pytest.mark.parametrize("kind,n", [("sphere", 2), ("sphere", 3), ("sphere", 4), ("sphere", 5), ("sphere", 6), ("sphere", 7),
                                     ("ellipsoid", 3), ("ellipsoid", 6), ("plane", 3), ("plane", 5)])
def test_analytic_fields_bit_exact(kind, n):
    """Lattice-aligned probes make exact zeros and ties common, so the arithmetic order matters."""
    rng = np.random.default_rng(n)
    if kind == "sphere":
        prod, orc = M.SphereManifold(np.zeros(n), 0.8), O.Field.sphere(np.zeros(n), 0.8)
    elif kind == "ellipsoid":
        c, a = rng.normal(size=n) * 0.1, rng.uniform(0.5, 1.0, size=n)
        prod, orc = M.EllipsoidManifold(c, a), O.Field.ellipsoid(c, a)
    else:
        nrm = rng.normal(size=n)
        prod, orc = M.PlaneManifold(nrm, 0.1), O.Field.plane(nrm, 0.1)
    lattice_pts = rng.integers(-8, 9, size=(20000, n)) * 0.1
    random_pts = rng.normal(size=(20000, n))
    for pts in (lattice_pts, random_pts):
        want = orc.values(pts)
        got = prod.values(pts)
        if kind == "plane":       # BLAS matvec order is not part of the contract; signs must agree off zero
            assert np.allclose(got, want, rtol=0, atol=1e-14)
        else:
            assert np.array_equal(got, want)
            assert np.array_equal(prod.signs(pts), orc.signs(pts))


def test_bisection(golden):
    g = golden("backend")
    f = M.SphereManifold(np.zeros(3), 1.0)
    got = M.intersection_points_batch(f, g["bisect_a"], g["bisect_b"], 1e-9)
    assert np.array_equal(got, g["bisect_points"])
    one = M.intersection_point(f, g["bisect_a"][0], g["bisect_b"][0], 1e-9)
    assert np.array_equal(one, g["bisect_points"][0])
    with pytest.raises(ValueError):
        M.intersection_point(f, [0.0, 0, 0], [0.1, 0, 0], 1e-9)
    assert M.edge_intersects(f, [0.0, 0, 0], [2.0, 0, 0]) and not M.edge_intersects(f, [0.0, 0, 0], [0.5, 0, 0])
    # segments shorter than eps are never bisected: t = 0.5
    a = np.array([[1.0, 0.0, 0.0]]); b = a + 1e-12
    assert np.array_equal(M.intersection_points_batch(f, a, b, 1e-9, signs_a=[-1]), a + 0.5 * (b - a))
    assert M.intersection_points_batch(f, np.zeros((0, 3)), np.zeros((0, 3)), 1e-9).shape == (0, 3)
    # linear field: root at t = 0.25 (pkg/tests/test_acceptance.py:318-339)
    pl = M.PlaneManifold([1.0, 0.0], 0.25)
    p = M.intersection_point(pl, [0.0, 0.0], [1.0, 0.0], 1e-9)
    assert abs(p[0] - 0.25) < 1e-9


def test_bisection_learned(golden):
    g = golden("traces")
    tag = "kclf_n4"
    m, of = product_manifold(g, tag), oracle_field(g, tag)
    inp = trace_inputs(g, tag)
    base, mask = g[f"{tag}_edge_base"].astype(np.float64), g[f"{tag}_edge_mask"]
    steps = np.array([[(int(mm) >> d) & 1 for d in range(4)] for mm in mask], dtype=np.float64)
    a = base * inp["scale"] + np.asarray(inp["offset"])
    b = (base + steps) * inp["scale"] + np.asarray(inp["offset"])
    got = M.intersection_points_batch(m, a, b, 1e-9)
    want = O.intersection_points_batch(of, a, b, 1e-9)
    assert np.allclose(got, want, rtol=POINT_RTOL, atol=POINT_ATOL)
    assert np.allclose(got, g[f"{tag}_points"], rtol=POINT_RTOL, atol=POINT_ATOL)


# ---- tracer -------------------------------------------------------------------------------------------
@pytest.mark.parametrize("tag", ANALYTIC_TRACES + LEARNED_TRACES)
def test_trace_matches_reference(golden, tag):
    g = golden("traces")
    inp = trace_inputs(g, tag)
    res = T.trace(inp["seeds"], product_manifold(g, tag), product_cfg(inp))
    base, mask, sa = res.edges.arrays()
    assert np.array_equal(base, g[f"{tag}_edge_base"]), "edge set / admission order differs"
    assert np.array_equal(mask, g[f"{tag}_edge_mask"])
    st, want = res.stats, g[f"{tag}_stats"]
    assert [st.levels, st.seeds, st.visited_edges, st.field_evaluations, st.dropped_out_of_box, int(st.complete),
            int(st.closure_ok)] == list(want[:7])
    assert (-1 if st.polyline_closed is None else int(st.polyline_closed)) == int(want[7])
    names = ("locate_cells", "cell_edges", "edge_cofaces", "coface_partner")
    stages = np.array([[names.index(s.name), s.level, s.items, s.capacity, s.produced] for s in st.stages])
    assert np.array_equal(stages, g[f"{tag}_stages"])
    adj = np.asarray(res.adjacency, dtype=np.int64).reshape(-1, 2)
    if f"{tag}_adjacency" in g:
        assert np.array_equal(adj, g[f"{tag}_adjacency"])
    else:
        digest = [adj.shape[0], int(adj[:, 0].sum()), int(adj[:, 1].sum()), int((adj[:, 0] * 31 + adj[:, 1]).sum() % (1 << 61))]
        assert digest == list(g[f"{tag}_adjacency_digest"])
    if tag.startswith("kclf"):
        assert np.allclose(res.points, g[f"{tag}_points"], rtol=POINT_RTOL, atol=POINT_ATOL)
    else:
        assert np.array_equal(res.points, g[f"{tag}_points"])
    # list-like behaviour of the lazy edge view
    assert len(res.edges) == st.visited_edges
    e0 = res.edges[0]
    assert isinstance(e0, L.PermSimplex) and e0.base == tuple(int(v) for v in base[0])
    e0.validate()


def test_locate_and_expand_api(golden):
    g = golden("traces")
    inp = trace_inputs(g, "sphere_n3")
    f, cfg = product_manifold(g, "sphere_n3"), product_cfg(inp)
    of = oracle_field(g, "sphere_n3")
    frontier = T.locate_edges(inp["seeds"], f, cfg)
    ot = O.Trace(of, 3, inp["scale"], inp["offset"])
    entries = ot.locate(inp["seeds"])
    assert [(e.base, e.parts) for e in frontier.edges] == [e for e, _ in entries]
    assert list(frontier.signs) == [s for _, s in entries]
    assert frontier.capacity == len(inp["seeds"]) * 6
    visited = set(frontier.edges)
    nxt = T.expand_frontier(frontier, visited, f, cfg)
    for e, s in entries:
        ot.admit(e, s)
    want = ot.expand(entries)
    assert [(e.base, e.parts) for e in nxt.edges] == [e for e, _ in want]
    assert visited == set(frontier.edges) | set(nxt.edges)
    with pytest.raises(ValueError):
        T.trace(np.zeros((0, 3)), f, cfg)
    with pytest.raises(ValueError):
        T.trace(np.zeros((1, 2)), f, cfg)
    with pytest.raises(ValueError):
        T.trace(inp["seeds"], f, T.TraceConfig(L.LatticeConfig(3, 0.5), box=((0, 0, 0), (1, 0, 1))))
    with pytest.raises(ValueError):
        T.trace(inp["seeds"], M.SphereManifold(np.zeros(2), 1.0), cfg)
    # a seed whose cell does not touch the zero set: explicit empty result
    empty = T.trace(np.array([[5.0, 5.0, 5.0]]), f, cfg)
    assert len(empty.edges) == 0 and empty.points.shape == (0, 3) and not empty.closure_ok and empty.adjacency == []


def test_trace_independent_of_seed_order_as_a_set(golden):
    g = golden("traces")
    inp = trace_inputs(g, "kclf_n4")
    m, cfg = product_manifold(g, "kclf_n4"), product_cfg(inp)
    a = T.trace(inp["seeds"], m, cfg)
    b = T.trace(inp["seeds"][::-1], m, cfg)
    ka = {(tuple(r), int(mm)) for r, mm in zip(*a.edges.arrays()[:2])}
    kb = {(tuple(r), int(mm)) for r, mm in zip(*b.edges.arrays()[:2])}
    assert ka == kb and a.closure_ok and b.closure_ok


# ---- coarse cells + refine ------------------------------------------------------------------------------
@pytest.mark.parametrize("tag", ["kclf_n3", "kclf_n4", "kclf_n5"])
def test_coarse_cells(golden, tag):
    g = golden("traces")
    inp = trace_inputs(g, tag)
    res = T.trace(inp["seeds"], product_manifold(g, tag), product_cfg(inp))
    cells = S.coarse_cells(res)
    base, perm = cells.arrays()
    if f"{tag}_cells_base" in g:
        assert np.array_equal(base, g[f"{tag}_cells_base"]) and np.array_equal(perm, g[f"{tag}_cells_perm"])
        c0 = cells[0]
        assert c0.dim == inp["n"] and c0.parts[-1] == (inp["n"],)
    else:
        n = inp["n"]
        assert len(cells) == int(g[f"{tag}_cells_count"][0])
        assert [int(base.sum()), int((perm.astype(np.int64) * np.arange(1, n + 1)).sum())] == list(g[f"{tag}_cells_digest"])
        keys = [tuple(b) + tuple(p) for b, p in zip(base.tolist(), perm.tolist())]
        assert keys == sorted(keys)


@pytest.mark.parametrize("tag", ["sphere_n2_k3", "sphere_n3_k2", "sphere_n4_k2"])
def test_refine_analytic(golden, tag):
    g = golden("refine")
    n, lam, k = g[f"{tag}_params"]
    n, k = int(n), int(k)
    f = M.SphereManifold(np.zeros(n), 0.8)
    cfg = T.TraceConfig(L.LatticeConfig(n, lam * k))
    res = T.trace(f.seed_point()[None, :], f, cfg)
    cells = S.coarse_cells(res)
    base, perm = cells.arrays()
    assert np.array_equal(base, g[f"{tag}_cells_base"]) and np.array_equal(perm, g[f"{tag}_cells_perm"])
    template = S.build_template(n, k)
    out = S.refine(cells, template, f, lambda p: p[:, 0] > 0.1, cfg)
    want = g[f"{tag}_points"]
    assert out.points.shape == want.shape
    if k == 2:
        assert np.array_equal(out.points, want)       # same dyadic bisection on bit-identical endpoints
    else:
        assert np.allclose(out.points, want, rtol=POINT_RTOL, atol=1e-12)
    assert np.array_equal(out.in_collision, g[f"{tag}_labels"])
    assert sum(b.crossing_edges for b in out.batch_stats) == int(g[f"{tag}_crossings"][0])
    assert np.array_equal(out.free_points, out.points[~out.in_collision])
    # same result from an explicit list of PermSimplex cells (host upload path) and under a tight budget
    again = S.refine(list(cells), template, f, lambda p: p[:, 0] > 0.1, cfg, memory_budget=7 * S._cell_bytes(template))
    assert np.array_equal(again.points, out.points) and np.array_equal(again.in_collision, out.in_collision)
    assert len(again.batch_stats) == -(-len(cells) // 7)
    assert sum(b.new_points for b in again.batch_stats) == out.points.shape[0]


def test_refine_learned_device_checker(golden):
    g = golden("traces")
    tag, n = "kclf_n3", 3
    inp = trace_inputs(g, tag)
    m, cfg = product_manifold(g, tag), product_cfg(inp)
    res = T.trace(inp["seeds"], m, cfg)
    cells = S.coarse_cells(res)
    rd, sd = robot_scene_dicts(n, 3)

    class Prob:
        robot, scene = CO.robot_from_dict(rd), CO.scene_from_dict(sd)

    template = S.build_template(n, 2)
    budget = int(g[f"{tag}_refine_budget"][0])
    out = S.refine(cells, template, m, P.not_free_checker(Prob), cfg, memory_budget=budget)
    want = g[f"{tag}_refine_points"]
    assert out.points.shape == want.shape
    assert np.allclose(out.points, want, rtol=POINT_RTOL, atol=POINT_ATOL)
    assert np.array_equal(out.in_collision, g[f"{tag}_refine_labels"])
    assert out.eps_dedup == float(g[f"{tag}_refine_eps_dedup"][0])
    rows = np.array([[b.cells, b.fine_vertices, b.crossing_edges, b.new_points] for b in out.batch_stats])
    assert np.array_equal(rows, g[f"{tag}_refine_batches"])
    # host-callable checker path gives the same labels
    host = S.refine(cells, template, m, lambda p: P.not_free_checker(Prob)(p), cfg)
    assert np.array_equal(host.points, out.points) and np.array_equal(host.in_collision, out.in_collision)
    # a failing checker is wrapped (pkg/tests/test_subdivision.py:262-270)
    def broken(p):
        raise RuntimeError("boom")
    with pytest.raises(S.RefineError, match="batch 0"):
        S.refine(cells, template, m, broken, cfg)
    with pytest.raises(S.RefineError, match="shape"):
        S.refine(cells, template, m, lambda p: np.zeros(3, dtype=bool), cfg)
    with pytest.raises(S.BudgetError):
        S.refine(cells, template, m, broken, cfg, memory_budget=10)
    empty = S.refine([], template, m, broken, cfg)
    assert empty.points.shape == (0, n) and empty.batch_stats == []


def test_refine_vs_oracle_4d_subset(golden):
    """4-D learned manifold, first 300 sorted cells: full oracle refine (eps-dedup included)."""
    g = golden("traces")
    tag, n = "kclf_n4", 4
    inp = trace_inputs(g, tag)
    m, cfg, of = product_manifold(g, tag), product_cfg(inp), oracle_field(g, tag)
    cells = [L.PermSimplex(tuple(int(v) for v in b), tuple((int(p),) for p in perm) + ((n,),))
             for b, perm in zip(g[f"{tag}_cells_base"][:300], g[f"{tag}_cells_perm"][:300])]
    rd, sd = robot_scene_dicts(n, 3)
    robot, scene = oracle_model(rd, sd)

    class Prob:
        robot_, scene_ = None, None
    Prob.robot, Prob.scene = CO.robot_from_dict(rd), CO.scene_from_dict(sd)
    out = S.refine(cells, S.build_template(n, 2), m, P.not_free_checker(Prob), cfg)
    ocells = [(c.base, c.parts) for c in cells]
    want = O.refine(ocells, O.build_template(n, 2), of, lambda p: O.not_free(robot, scene, p), inp["scale"],
                    inp["offset"], 2, inp["eps"])
    assert out.points.shape == want["points"].shape
    assert np.allclose(out.points, want["points"], rtol=POINT_RTOL, atol=POINT_ATOL)
    assert np.array_equal(out.in_collision, want["in_collision"])
    assert sum(b.crossing_edges for b in out.batch_stats) == sum(want["crossing_edges"])


# ---- refine / eps-dedup / labels at n = 5 and n = 6 (the benchmarked dimension) -------------------------------------
def _cells_sha(cb, cp):
    import hashlib
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(cb, dtype=np.int16).tobytes())
    h.update(np.ascontiguousarray(cp, dtype=np.uint8).tobytes())
    return h.hexdigest()


def _device_problem(n, nobs):
    rd, sd = robot_scene_dicts(n, nobs)

    class Prob:
        robot, scene = CO.robot_from_dict(rd), CO.scene_from_dict(sd)
    return Prob, oracle_model(rd, sd)


@pytest.mark.parametrize("tag", ["kclf_n5", "kclf_n6"])
def test_refine_high_dim_vs_reference(golden, tag):
    """The REAL reference's refine (tests/golden/refine_hd.npz, generated by make_golden.py) of the first / middle /
    last runs of sorted coarse cells at n = 5 and n = 6, one cell per batch: per-cell crossing counts, per-cell fresh
    points of the greedy eps-dedup (3^n neighbour buckets, order-dependent: SURVEY hard part 3), kept points in the
    reference's order, collision labels (8 primitives incl. cylinders and spheres).  subdivision.py:195-217, :256-278."""
    g, gh = golden("traces"), golden("refine_hd")
    inp = trace_inputs(g, tag)
    n = inp["n"]
    m, cfg = product_manifold(g, tag), product_cfg(inp)
    cells = L.cells_from_arrays(gh[f"{tag}_sub_base"].astype(np.int32), gh[f"{tag}_sub_perm"])
    Prob, _ = _device_problem(n, 8)
    template = S.build_template(n, 2)
    out = S.refine(cells, template, m, P.not_free_checker(Prob), cfg, memory_budget=S._cell_bytes(template))
    rows = np.array([[b.crossing_edges, b.new_points] for b in out.batch_stats])
    assert np.array_equal(rows, gh[f"{tag}_sub_per_cell"])
    want = gh[f"{tag}_sub_points"]
    assert out.points.shape == want.shape
    assert np.allclose(out.points, want, rtol=POINT_RTOL, atol=POINT_ATOL)
    assert np.array_equal(out.in_collision, gh[f"{tag}_sub_labels"])
    assert out.eps_dedup == float(gh[f"{tag}_sub_eps_dedup"][0])
    # the same cells inside the full job: every kept point of the subset run that the full run also keeps sits at
    # the same place; the full run's cell list equals the reference's (sha256 over the sorted (base, perm) arrays)
    res = T.trace(inp["seeds"], m, cfg)
    full = S.coarse_cells(res)
    cb, cp = full.arrays()
    assert len(full) == int(gh[f"{tag}_cells_count"][0])
    assert _cells_sha(cb, cp) == str(gh[f"{tag}_cells_sha256"][0])
    pick = gh[f"{tag}_pick"]
    assert np.array_equal(cb[pick], gh[f"{tag}_sub_base"]) and np.array_equal(cp[pick], gh[f"{tag}_sub_perm"])


@pytest.mark.parametrize("workload,run", [("dof5", 90), ("dof6", 70)])
def test_refine_bench_workloads_vs_oracle(workload, run):
    """The bench workloads themselves (dof5: cylinders + spheres; dof6: the headline config): first / middle / last runs
    of the sorted coarse cells refined on the CUDA path and by the oracle, one cell per batch."""
    from bench import build_workload
    wl = build_workload(workload)
    a = wl.arrays
    res = T.trace(wl.seeds, wl.manifold, wl.cfg)
    cells = S.coarse_cells(res)
    cb, cp = cells.arrays()
    mid = len(cells) // 2
    pick = np.r_[0:run, mid - run // 2:mid - run // 2 + run, len(cells) - run:len(cells)]
    sub = L.cells_from_arrays(cb[pick], cp[pick])
    checker = P.not_free_checker(wl.problem)
    out = S.refine(sub, wl.template, wl.manifold, checker, wl.cfg, memory_budget=S._cell_bytes(wl.template))
    scale, gain, lo, hi = a.barrier
    of = O.Field.rbf(a.support, a.weights, a.gamma, a.bias, barrier=(scale, gain, lo, hi))
    robot, scene = oracle_model(a.robot_dict, a.scene_dict)
    O.THREADS = min(os.cpu_count() or 1, 16)
    try:
        want = O.refine([(c.base, c.parts) for c in sub], O.build_template(a.n, a.k), of,
                        lambda p: O.not_free(robot, scene, p), a.coarse, np.zeros(a.n), a.k, a.eps, batch_cells=1)
    finally:
        O.THREADS = 1
    rows = np.array([[b.crossing_edges, b.new_points] for b in out.batch_stats])
    assert np.array_equal(rows[:, 0], want["crossing_edges"]) and np.array_equal(rows[:, 1], want["new_points"])
    assert rows[:, 0].sum() > 20 * run
    assert out.points.shape == want["points"].shape
    assert np.allclose(out.points, want["points"], rtol=POINT_RTOL, atol=POINT_ATOL)
    assert np.array_equal(out.in_collision, want["in_collision"])
    # the capped oracle BFS reproduces the head of the device's ordered edge list (admission order, tracer.py:359-375)
    cap = 1500
    tr = O.Trace(of, a.n, a.coarse, None, a.box, cap, a.eps).run(a.seeds)
    base, mask, _ = res.edges.arrays()
    ob = np.array([e[0] for e in tr.edges]); om = np.array([sum(1 << d for d in e[1][0]) for e in tr.edges])
    assert len(tr.edges) == cap and np.array_equal(ob, base[:cap]) and np.array_equal(om, mask[:cap])


# ---- collision ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("n,nobs", [(3, 3), (4, 3), (5, 8), (6, 8)])
def test_collision(golden, n, nobs):
    g = golden("collision")
    rd, sd = robot_scene_dicts(n, nobs)
    robot, scene = CO.robot_from_dict(rd), CO.scene_from_dict(sd)
    q = g[f"coll_n{n}_q"]
    got = CO.batch_check(q, robot, scene, on_limit="unfree")
    assert got.dtype == bool and np.array_equal(got, g[f"coll_n{n}_unfree"])
    inside = np.all(np.abs(q) <= 1.5, axis=1)
    assert np.array_equal(CO.batch_check(q[inside], robot, scene), g[f"coll_n{n}_hits_inside"])
    assert np.allclose(CO.fk_batch(robot, q[:40]), g[f"coll_n{n}_fk"], rtol=0, atol=1e-13)
    bad = int(np.nonzero(~inside)[0][0])
    with pytest.raises(CO.LimitError, match=f"configuration {bad} "):
        CO.batch_check(q, robot, scene)
    row = q[inside][0]
    assert CO.config_in_collision(row, robot, scene) == bool(g[f"coll_n{n}_hits_inside"][0])
    assert CO.batch_check(np.zeros((0, n)), robot, scene).shape == (0,)
    # permutation equivariance and batch-size irrelevance (pkg/tests/test_collision.py)
    perm = np.random.default_rng(0).permutation(int(inside.sum()))
    assert np.array_equal(CO.batch_check(q[inside][perm], robot, scene, batch_size=17), g[f"coll_n{n}_hits_inside"][perm])


def test_collision_prismatic_posed_and_first_contact(golden):
    g = golden("collision")
    robot, scene = CO.robot_from_dict(PRISM_ROBOT), CO.scene_from_dict(PRISM_SCENE)
    q = g["coll_prism_q"]
    hits = CO.batch_check(q, robot, scene)
    assert np.array_equal(hits, g["coll_prism_hits"])
    assert np.allclose(CO.fk_batch(robot, q[:40]), g["coll_prism_fk"], rtol=0, atol=1e-13)
    i_hit, i_free = int(np.nonzero(hits)[0][0]), int(np.nonzero(~hits)[0][0])
    rep = CO.first_contact(q[i_hit], robot, scene)
    assert rep.hit and rep.sphere_index is not None and rep.obstacle_index is not None
    assert not CO.first_contact(q[i_free], robot, scene).hit
    with pytest.raises(CO.LimitError):
        CO.forward_kinematics(robot, [5.0, 0.0])
    with pytest.raises(ValueError):
        CO.forward_kinematics(robot, [np.nan, 0.0])
    box = scene.obstacles[2]
    centre = box.pose.translation + box.pose.rotation @ np.array([0.15 + 0.05, 0.0, 0.0])
    assert CO.sphere_box_collides(centre, 0.05 + 1e-9, box) and not CO.sphere_box_collides(centre, 0.05 - 1e-9, box)


def test_collision_vs_distance_oracle():
    """10^5 random sphere-vs-box / cylinder cases against closed-form distances, skipping |gap| <= 1e-12
    (pkg/tests/test_acceptance.py:227-260)."""
    rng = np.random.default_rng(42)
    c = rng.uniform(-2, 2, size=(100000, 3)); r = rng.uniform(0.01, 0.8, size=100000)
    h = np.array([0.6, 0.35, 0.9])
    d = np.maximum(np.abs(c) - h, 0.0)
    gap = np.linalg.norm(d, axis=1) - r
    got = B.sphere_box_hits(c, r, *(2 * h)).astype(bool)
    keep = np.abs(gap) > 1e-12
    assert np.array_equal(got[keep], (gap <= 0)[keep])
    dz = np.maximum(np.abs(c[:, 2]) - 0.5, 0.0); dr = np.maximum(np.hypot(c[:, 0], c[:, 1]) - 0.4, 0.0)
    gap = np.hypot(dz, dr) - r
    got = B.sphere_cylinder_hits(c, r, 1.0, 0.4).astype(bool)
    keep = np.abs(gap) > 1e-12
    assert np.array_equal(got[keep], (gap <= 0)[keep])


# ---- full-size properties (BASELINE config shapes; no CPU oracle can follow at this size) --------------------
def test_dof6_full_size_properties():
    from bench import build_workload
    wl = build_workload("dof6")
    res = T.trace(wl.seeds, wl.manifold, wl.cfg)
    st = res.stats
    assert st.closure_ok and st.dropped_out_of_box == 0 and st.complete
    # the reference finds 47 594 edges / 8 677 vertex evaluations on this recipe
    # (vertex evaluations also count the seed cells' own corners, so they vary with the seed draw)
    assert st.visited_edges == 47594 and 8677 - 140 <= st.field_evaluations <= 8677 + 140
    base, mask, sa = res.edges.arrays()
    # every traced edge is sign-changing under an independent evaluation of its endpoints
    steps = ((mask[:, None] >> np.arange(6)) & 1).astype(np.float64)
    a = base * wl.cfg.lattice.scale + np.asarray(wl.cfg.lattice.offset)
    b = (base + steps) * wl.cfg.lattice.scale + np.asarray(wl.cfg.lattice.offset)
    s_a, s_b = wl.manifold.signs(a), wl.manifold.signs(b)
    assert np.array_equal(s_a, sa) and np.all(s_a != s_b)
    # no duplicates, and each point sits inside an eps bracket on its own edge
    assert len({(tuple(r), int(m)) for r, m in zip(base.tolist(), mask.tolist())}) == len(mask)
    t = np.einsum("ij,ij->i", res.points - a, b - a) / np.einsum("ij,ij->i", b - a, b - a)
    assert np.all((t > 0) & (t < 1))
    assert np.allclose(res.points, a + t[:, None] * (b - a), atol=1e-12)
    # adjacency: every crossing 2-face has exactly two crossing edges -> each edge has as many partners as cofaces
    adj = np.asarray(res.adjacency)
    deg = np.bincount(adj.ravel(), minlength=len(mask))
    pc = np.array([bin(int(m)).count("1") for m in mask])
    assert np.array_equal(deg, (2 ** pc - 2) + (2 ** (7 - pc) - 2))
    cells = S.coarse_cells(res)
    cb, cp = cells.arrays()
    keys = np.concatenate([cb.astype(np.int64), cp.astype(np.int64)], axis=1)
    order = np.lexsort(keys.T[::-1])
    assert np.array_equal(order, np.arange(len(order)))       # sorted, hence unique
    assert len(cells) > 10 * st.visited_edges


def test_dof6_full_size_refine_properties(monkeypatch):
    """BASELINE-size refinement (1.3 M cells, 50.8 M crossings): the fast root-solve path (tensor-core screen, enclosure
    Newton, replay) must return the SAME points as plain fp64 bisection on the same device, every point must be an
    eps-accurate zero of the field, and the result must not depend on how the cells are sliced over ranks."""
    import torch
    from bench import build_workload
    from paper_2406_04795_b200.distributed import CudaEngine, cell_slice
    out = {}
    for mode in ("1", "0", "1-two-groups"):
        monkeypatch.setenv("PERMATRACE_B200_PRECISION", mode[0])
        monkeypatch.setenv("PERMATRACE_B200_TC4", "0" if mode == "1-two-groups" else "1")
        wl = build_workload("dof6")
        checker = P.not_free_checker(wl.problem)
        res = T.trace(wl.seeds, wl.manifold, wl.cfg)
        ref = S.refine(S.coarse_cells(res), wl.template, wl.manifold, checker, wl.cfg)
        out[mode] = (res.points.copy(), ref.points.copy(), ref.in_collision.copy(), sum(b.crossing_edges for b in ref.batch_stats))
        if mode == "1":
            # three virtual ranks: slices refined separately, merged in rank order, deduplicated once
            eng = CudaEngine(wl.manifold, wl.cfg, wl.template, checker)
            info = eng.trace(torch.from_numpy(wl.seeds).cuda())
            parts = [eng.candidates(*cell_slice(info["cells"], r, 3)) for r in range(3)]
            merged = torch.cat([p for p, _ in parts], dim=0)
            kept, labels = eng.dedup_label(merged)
            assert np.array_equal(merged[kept].cpu().numpy(), ref.points)
            assert np.array_equal(labels.cpu().numpy().astype(bool), ref.in_collision)
            assert sum(c for _, c in parts) == out[mode][3]
            # zero-set accuracy on a sample: |F| <= 4 eps (|grad F| + 1e-12)   (reference pipeline.py:519-526)
            from paper_2406_04795_b200.pipeline import _gradient_norms
            sample = ref.points[:: max(1, ref.points.shape[0] // 20000)]
            resid = np.abs(wl.manifold.values(sample))
            assert np.all(resid <= 4.0 * wl.cfg.eps * (_gradient_norms(wl.manifold, sample) + 1e-12))
    fast, slow = out["1"], out["0"]
    assert fast[3] == slow[3] == 50766688
    assert fast[0].shape == slow[0].shape and fast[1].shape == slow[1].shape == (1606495, 6)
    assert np.max(np.abs(fast[0] - slow[0])) <= 1e-8 and np.max(np.abs(fast[1] - slow[1])) <= 1e-8
    assert np.array_equal(fast[2], slow[2])
    # the four-group and the two-group tensor-core screens only differ in which signs fp32 manages to prove
    two = out["1-two-groups"]
    assert two[3] == fast[3] and two[1].shape == fast[1].shape
    assert np.max(np.abs(fast[0] - two[0])) <= 1e-8 and np.max(np.abs(fast[1] - two[1])) <= 1e-8
    assert np.array_equal(fast[2], two[2])


# ---- device pipeline and the sharded driver on one GPU -----------------------------------------------------
def test_device_pipeline_and_sharded_driver_agree_with_public_api(golden):
    from paper_2406_04795_b200 import engine
    from paper_2406_04795_b200.distributed import CudaEngine, ShardedProof
    import torch
    g = golden("traces")
    tag, n = "kclf_n4", 4
    inp = trace_inputs(g, tag)
    m, cfg = product_manifold(g, tag), product_cfg(inp)
    rd, sd = robot_scene_dicts(n, 3)

    class Prob:
        robot, scene = CO.robot_from_dict(rd), CO.scene_from_dict(sd)

    checker = P.not_free_checker(Prob)
    template = S.build_template(n, 2)
    res = T.trace(inp["seeds"], m, cfg)
    ref = S.refine(S.coarse_cells(res), template, m, checker, cfg)
    seeds = torch.from_numpy(inp["seeds"]).cuda()
    counts = engine.DevicePipeline(m, cfg, template, checker).step(seeds.data_ptr(), seeds.shape[0])
    assert counts["trace_edges"] == len(res.edges) and counts["points"] == ref.points.shape[0]
    assert counts["crossing_edges"] == sum(b.crossing_edges for b in ref.batch_stats)
    assert counts["free_points"] == int((~ref.in_collision).sum())
    out = ShardedProof(CudaEngine(m, cfg, template, checker)).run(seeds)
    assert np.array_equal(out["points"].cpu().numpy(), ref.points)
    assert np.array_equal(out["in_collision"].cpu().numpy(), ref.in_collision)
    assert out["crossing_edges"] == counts["crossing_edges"] and out["cells"] == counts["cells"]
    # two "virtual ranks" on one device: slices merged by hand reproduce the same result
    eng = CudaEngine(m, cfg, template, checker)
    info = eng.trace(seeds)
    from paper_2406_04795_b200.distributed import cell_slice
    parts = [eng.candidates(*cell_slice(info["cells"], r, 3)) for r in range(3)]
    merged = torch.cat([p for p, _ in parts], dim=0)
    kept, labels = eng.dedup_label(merged)
    assert np.array_equal(merged[kept].cpu().numpy(), ref.points)
    assert np.array_equal(labels.cpu().numpy().astype(bool), ref.in_collision)
    assert sum(c for _, c in parts) == counts["crossing_edges"]


# ---- tensor-core screen: calibration of the exponent error bound -----------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["kclf_n4", "kclf_n6"])
def test_tc_screen_exponent_error(golden, tag):
    """|exponent on the tensor cores - fp64 exponent| over random segment midpoints, in units of
    2^-24 * gamma*log2e*(|p|+max|s|)^2, must stay below half of PT_TC_ARG_ULPS = 16 (csrc/pt_field.cuh)."""
    import ctypes as C
    from paper_2406_04795_b200 import _cabi
    g = golden("traces")
    inp = trace_inputs(g, tag)
    manifold = product_manifold(g, tag)
    rng = np.random.default_rng(7)
    m = 50_000
    lo, hi = np.asarray(inp["box"][0]), np.asarray(inp["box"][1])
    a = rng.uniform(lo, hi, size=(m, inp["n"]))
    b = a + rng.normal(scale=0.3, size=a.shape)
    out = np.zeros(m)
    rc = _cabi.lib.pt_debug_tc_arg_error(_cabi.context().handle, manifold.device_field(), a.ctypes.data, b.ctypes.data, m, out.ctypes.data)
    _cabi.check(rc)
    assert np.isfinite(out).all() and 0.0 < out.max() < 8.0


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["kclf_n4", "kclf_n6"])
def test_tc_sign_evaluation_equals_fp64_signs(golden, tag):
    """Large sign batches run on the tensor cores with an FP64 recheck of every unproven row: the signs must equal
    those of the FP64 values, including at points ON the zero set (the golden intersection points) and within
    1e-12 .. 1e-6 of it."""
    g = golden("traces")
    inp = trace_inputs(g, tag)
    manifold = product_manifold(g, tag)
    rng = np.random.default_rng(11)
    lo, hi = np.asarray(inp["box"][0]), np.asarray(inp["box"][1])
    on = g[f"{tag}_points"]
    near = np.concatenate([on + rng.normal(scale=s, size=on.shape) for s in (0.0, 1e-12, 1e-9, 1e-6)])
    pts = np.concatenate([rng.uniform(lo, hi, size=(30_000, inp["n"])), near])
    values = manifold.values(pts)
    signs = manifold.signs(pts)
    assert signs.shape == (pts.shape[0],) and set(np.unique(signs)) <= {-1, 1}
    assert np.array_equal(signs, np.where(values > 0.0, 1, -1))


def test_learned_field_gradient(golden):
    """KernelClassifierManifold.gradient(s) on the device against the reference formula (manifold.py:210-217),
    and against central differences of the device values."""
    g = golden("traces")
    for tag in ("kclf_n3", "kclf_n6"):
        inp = trace_inputs(g, tag)
        m = product_manifold(g, tag)
        rng = np.random.default_rng(3)
        lo, hi = np.asarray(inp["box"][0]), np.asarray(inp["box"][1])
        pts = rng.uniform(lo, hi, size=(257, inp["n"]))
        got = m.gradients(pts)
        d = pts[:, None, :] - m.support[None, :, :]
        kern = np.exp(-m.gamma * np.einsum("ijk,ijk->ij", d, d)) * m.weights[None, :]
        want = -2.0 * m.gamma * np.einsum("ij,ijk->ik", kern, d) - np.stack([m.barrier.gradient(q) for q in pts])
        scale = np.abs(kern).sum(axis=1, keepdims=True) * 2.0 * m.gamma * 8.0
        assert np.all(np.abs(got - want) <= 1e-12 * scale + 1e-12)
        assert np.allclose(m.gradient(pts[5]), got[5], rtol=0, atol=0)
        h = 1e-6
        for dim in range(inp["n"]):
            e = np.zeros(inp["n"]); e[dim] = h
            fd = (m.values(pts[:16] + e) - m.values(pts[:16] - e)) / (2 * h)
            assert np.allclose(fd, got[:16, dim], rtol=1e-5, atol=1e-6 * float(scale.max()))


def test_collision_fp32_screen_equals_fp64(monkeypatch):
    """Large batches go through the fp32 screen (certain hit / certain miss / undecided -> fp64 kernel): the masks
    must equal the plain fp64 kernel's on random configurations, on configurations dragged onto obstacle surfaces
    (bisected along segments between a free and a colliding configuration), and on out-of-limit rows."""
    from tests.conftest import robot_scene_dicts
    for n, nobs in ((6, 8), (4, 3)):
        rd, sd = robot_scene_dicts(n, nobs)
        rng = np.random.default_rng(5)
        q = rng.uniform(-1.6, 1.6, size=(60_000, n))            # limits are +-1.5: some rows are outside
        masks = {}
        for mode in ("0", "1"):
            monkeypatch.setenv("PERMATRACE_B200_PRECISION", mode)
            robot, scene = CO.robot_from_dict(rd), CO.scene_from_dict(sd)
            masks[mode] = CO.batch_check(q, robot, scene, on_limit="unfree")
            if mode == "0":
                # touching configurations: bisect free/colliding pairs with the fp64 kernel to ~1e-9 of the surface
                inside = np.all(np.abs(q) <= 1.5, axis=1)
                free = q[inside & ~masks["0"]][:4000]
                coll = q[inside & masks["0"]][:4000]
                k = min(len(free), len(coll))
                a, b = free[:k].copy(), coll[:k].copy()
                for _ in range(30):
                    mid = 0.5 * (a + b)
                    hit = CO.batch_check(mid, robot, scene, on_limit="unfree")
                    b[hit], a[~hit] = mid[hit], mid[~hit]
                near = np.concatenate([a, b, 0.5 * (a + b)])
                near = np.concatenate([near, near + rng.normal(scale=1e-6, size=near.shape)])
                masks["near0"] = CO.batch_check(near, robot, scene, on_limit="unfree")
            else:
                masks["near1"] = CO.batch_check(near, robot, scene, on_limit="unfree")
        assert masks["0"].sum() > 1000 and (~masks["0"]).sum() > 1000
        assert np.array_equal(masks["0"], masks["1"])
        assert near.shape[0] >= 4096 and np.array_equal(masks["near0"], masks["near1"])


def test_large_support_set_fallback_paths(monkeypatch):
    """S = 4096 support vectors do not fit one CTA's shared memory: the root solve then uses the SIMT fp32 screen and the
    tiled rest kernel.  Fast path == plain fp64 bisection on the same device, and the trace is unchanged."""
    from paper_2406_04795_b200.scenes import synthetic_support
    from bench import _train_numpy
    n, lam, k = 4, 0.3, 2
    pos, neg, rng = synthetic_support(n, 4096, 0.9, 1.5, seed=3)
    support, weights = _train_numpy(pos, neg, 2.0, 1e-3)
    sigma = 0.5
    lo, hi = -1.5 * np.ones(n), 1.5 * np.ones(n)
    coarse = lam * k
    margin = max(3.0 * coarse, 2.0 * sigma + (1.0 + 2.0 * np.sqrt(n)) * coarse)
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("PERMATRACE_B200_PRECISION", mode)
        m = M.KernelClassifierManifold(support, weights, 2.0, lam * 2.0, barrier=M.BoxBarrier(lo, hi, sigma / 4.0, 2.0 / sigma))
        cfg = T.TraceConfig(L.LatticeConfig(n, coarse), box=(tuple(lo - margin), tuple(hi + margin)), eps=1e-9)
        seeds = M.sample_seeds(m, (lo, hi), 12, rng=np.random.default_rng(1), min_separation=coarse / 2.0)
        res = T.trace(seeds, m, cfg)
        ref = S.refine(S.coarse_cells(res), S.build_template(n, k), m, lambda p: np.zeros(len(p), dtype=bool), cfg)
        out[mode] = (res.edges.arrays(), res.points.copy(), ref.points.copy(), res.stats.closure_ok)
    assert out["1"][3] and out["0"][3]
    for a, b in zip(out["0"][0], out["1"][0]):
        assert np.array_equal(a, b)
    assert out["0"][1].shape == out["1"][1].shape and out["0"][2].shape == out["1"][2].shape and out["1"][2].shape[0] > 4096
    assert np.max(np.abs(out["0"][1] - out["1"][1])) <= 1e-8 and np.max(np.abs(out["0"][2] - out["1"][2])) <= 1e-8


@pytest.mark.gpu
def test_ill_conditioned_field_root_solve(monkeypatch):
    """Barely regularised ridge weights (sum|w| ~ 10^5 x the field's scale): the fp32 screen proves next to nothing, so the
    root solve runs on its fp64 machinery alone -- resolve rounds instead of the screen, proof retries over shrinking
    lists, wide rows stepping inside the Newton kernel.  Same traced edges and the same points as plain fp64 bisection,
    up to the evaluation noise of such a field."""
    from paper_2406_04795_b200.scenes import synthetic_support
    from bench import _train_numpy
    n, lam, k = 4, 0.3, 2
    pos, neg, rng = synthetic_support(n, 2048, 0.9, 1.5, seed=5)
    support, weights = _train_numpy(pos, neg, 2.0, 1e-7)
    assert np.abs(weights).sum() > 1e4
    sigma = 0.5
    lo, hi = -1.5 * np.ones(n), 1.5 * np.ones(n)
    coarse = lam * k
    margin = max(3.0 * coarse, 2.0 * sigma + (1.0 + 2.0 * np.sqrt(n)) * coarse)
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("PERMATRACE_B200_PRECISION", mode)
        m = M.KernelClassifierManifold(support, weights, 2.0, lam * 2.0, barrier=M.BoxBarrier(lo, hi, sigma / 4.0, 2.0 / sigma))
        cfg = T.TraceConfig(L.LatticeConfig(n, coarse), box=(tuple(lo - margin), tuple(hi + margin)), eps=1e-9)
        seeds = M.sample_seeds(m, (lo, hi), 12, rng=np.random.default_rng(1), min_separation=coarse / 2.0)
        res = T.trace(seeds, m, cfg)
        ref = S.refine(S.coarse_cells(res), S.build_template(n, k), m, lambda p: np.zeros(len(p), dtype=bool), cfg,
                       eps_dedup=1e-12)
        out[mode] = (res.edges.arrays(), res.points.copy(), ref.points.copy(), res.stats.closure_ok)
    for a, b in zip(out["0"][0], out["1"][0]):
        assert np.array_equal(a, b)
    assert out["0"][1].shape == out["1"][1].shape and out["0"][2].shape == out["1"][2].shape and out["1"][2].shape[0] > 4096
    assert np.max(np.abs(out["0"][1] - out["1"][1])) <= 1e-7 and np.max(np.abs(out["0"][2] - out["1"][2])) <= 1e-7
    resid = np.abs(m.values(out["1"][2]))
    from paper_2406_04795_b200.pipeline import _gradient_norms
    assert np.all(resid <= 4.0 * 1e-9 * (_gradient_norms(m, out["1"][2]) + 1e-12) + 1e-9 * np.abs(weights).sum() * 1e-3)


# ---- one-pass Taylor-model root solve (pt_field_taylor.cuh) --------------------------------------------------
def _crossing_segments(m, lo, hi, count, step, rng, max_axes, generic_frac=0.0):
    """Random lattice-like segments (1..max_axes coordinates move by `step`, all by the same signed amount -- the rows the
    Taylor kernel groups by direction) whose end points have different signs; a fraction `generic_frac` of them gets an
    arbitrary direction of that length instead (rows that keep the N-term dot product)."""
    n = lo.size
    a_rows, b_rows, s_rows = [], [], []
    have = 0
    while have < count:
        a = rng.uniform(lo, hi, size=(4 * count, n))
        axes = rng.integers(1, max_axes + 1, size=a.shape[0])
        order = np.argsort(rng.random(a.shape), axis=1)                       # a random subset of `axes[i]` coordinates
        d = (order < axes[:, None]) * (step * rng.choice([-1.0, 1.0], size=(a.shape[0], 1)))
        if generic_frac > 0.0:
            g = rng.normal(size=a.shape)
            g *= (np.linalg.norm(d, axis=1) / np.linalg.norm(g, axis=1))[:, None]
            d = np.where(rng.random(a.shape[0])[:, None] < generic_frac, g, d)
        b = a + d
        sa, sb = m.signs(a), m.signs(b)
        keep = sa != sb
        a_rows.append(a[keep]); b_rows.append(b[keep]); s_rows.append(sa[keep].astype(np.int8))
        have += int(keep.sum())
    return np.concatenate(a_rows)[:count], np.concatenate(b_rows)[:count], np.concatenate(s_rows)[:count]


@pytest.mark.gpu
@pytest.mark.parametrize("n,S,step,gamma,reg", [(6, 2048, 0.175, 2.0, 1e-3), (4, 1500, 0.15, 2.0, 1e-3), (3, 700, 0.3, 1.0, 1e-3),
                                                (6, 4096, 0.175, 2.0, 1e-3), (5, 1024, 0.45, 2.0, 1e-5), (7, 512, 0.2, 1.5, 1e-3),
                                                (2, 300, 0.1, 3.0, 1e-3)])
def test_taylor_root_solve_equals_plain_bisection(monkeypatch, precision_mode, n, S, step, gamma, reg):
    """Large batches take the one-pass Taylor-model kernel.  Its brackets are the reference's dyadic brackets, so the points
    must be BIT-identical to plain fp64 bisection on the same device except where a visited midpoint is ambiguous -- |F| there
    below the reference's own cross-backend tolerance on the kernel sum -- and then end in the neighbouring cell (<= eps away).
    Well-conditioned fields (the n >= 5 cases) have no such rows; the small, densely sampled ones (n <= 4: sum|w| is 10^4..10^5
    times the field's scale) have a few per thousand in EVERY fp64 implementation."""
    if precision_mode != "fast":
        pytest.skip("compares the two modes itself")
    from paper_2406_04795_b200.scenes import synthetic_support
    from bench import _train_numpy
    pos, neg, rng = synthetic_support(n, S, 0.9 if n < 6 else 1.3, 1.5, seed=11 + n)
    support, weights = _train_numpy(pos, neg, gamma, reg)
    sigma = 1.0 / np.sqrt(2.0 * gamma)
    lo, hi = -1.5 * np.ones(n), 1.5 * np.ones(n)
    eps = 1e-9
    pts = {}
    left = [0]
    # ("1", "1"): the library's own choice at this batch size (generic kernel, one lane per edge); "grouped": the
    # direction-table kernel the big refinement batches take (grouping forced); "shared": generic kernel with four lanes per
    # edge (what tiny batches take)
    for mode, taylor in (("1", "1"), ("1", "grouped"), ("1", "shared"), ("0", "1"), ("1", "0")):
        monkeypatch.setenv("PERMATRACE_B200_PRECISION", mode)
        monkeypatch.setenv("PERMATRACE_B200_TAYLOR", "0" if taylor == "0" else "1")
        monkeypatch.delenv("PERMATRACE_B200_TAYLOR_GROUP_MIN", raising=False)
        monkeypatch.delenv("PERMATRACE_B200_TAYLOR_SHARE", raising=False)
        if taylor == "grouped":
            monkeypatch.setenv("PERMATRACE_B200_TAYLOR_GROUP_MIN", "1")
        if taylor == "shared":
            monkeypatch.setenv("PERMATRACE_B200_TAYLOR_SHARE", "4")
        m = M.KernelClassifierManifold(support, weights, gamma, 0.3 * np.sqrt(2.0 * gamma),
                                       barrier=M.BoxBarrier(lo, hi, sigma / 4.0, 2.0 / sigma))
        if not pts:
            # four fifths lattice edges (grouped by direction: direction-table kernel), one fifth arbitrary segments
            a, b, sa = _crossing_segments(m, lo - 0.3, hi + 0.3, 160_000, step, np.random.default_rng(n), min(n, 6), generic_frac=0.2)
        work = np.zeros(6, dtype=np.int64)
        _cabi.check(_cabi.lib.pt_ctx_work_counters(_cabi.context().handle, work.ctypes.data, 1))
        pts[(mode, taylor)] = M.intersection_points_batch(m, a, b, eps, signs_a=sa)
        _cabi.check(_cabi.lib.pt_ctx_work_counters(_cabi.context().handle, work.ctypes.data, 1))
        rows = int(_cabi.lib.pt_ctx_taylor_rows(_cabi.context().handle))
        assert rows == (len(a) if mode == "1" and taylor != "0" else 0)
        if rows:
            left[0] = int(work[3])
    new, plain, old = pts[("1", "1")], pts[("0", "1")], pts[("1", "0")]
    grouped, shared = pts[("1", "grouped")], pts[("1", "shared")]
    diff, seg2 = b - a, np.einsum("ij,ij->i", b - a, b - a)
    tol = 1e-12 * (np.abs(weights).sum() + abs(m.bias))        # the reference's own cross-backend tolerance on F
    for name, got in (("taylor", new), ("taylor grouped", grouped), ("taylor 4 lanes / edge", shared), ("screen+newton", old)):
        assert np.max(np.abs(got - plain)) <= 2.5e-9
        rows = np.flatnonzero(np.any(got != plain, axis=1))
        assert len(rows) <= len(a) // 200, f"{name}: {len(rows)} of {len(a)} rows differ from plain fp64 bisection"
        if len(rows):
            # the two bisections parted at the dyadic midpoint between their final cells: |F| there must be below the noise
            t1 = np.einsum("ij,ij->i", got[rows] - a[rows], diff[rows]) / seg2[rows]
            t0 = np.einsum("ij,ij->i", plain[rows] - a[rows], diff[rows]) / seg2[rows]
            tm = np.round(0.5 * (t0 + t1) * 2.0 ** 40) / 2.0 ** 40
            disputed = np.abs(m.values(a[rows] + tm[:, None] * diff[rows]))
            assert np.all(disputed <= tol), f"{name}: a differing row is not ambiguous: |F| = {disputed.max():.3g} > {tol:.3g}"
        print(f"{name} n={n} S={S}: {len(rows)} of {len(a)} rows differ from plain bisection (all ambiguous)")
    print(f"taylor n={n} S={S}: {left[0]} of {len(a)} rows left to the evaluation kernels")
