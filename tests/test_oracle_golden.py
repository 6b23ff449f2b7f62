"""Pin the CPU oracle against golden vectors produced by the real reference (make_golden.py).

Everything here runs on the CPU.  Integer / index results must match bit for bit; floating-point
results produced by the same numpy expressions on the same image must match exactly too, except
the kernel sum, where the reference's own backend tolerance applies
(pkg/tests/test_backends.py:81-93: 1e-12 * (sum|w| + |bias|)).
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import permatrace_oracle as O
from tests.conftest import (ANALYTIC_TRACES, LEARNED_TRACES, PRISM_ROBOT, PRISM_SCENE, analytic_spec, mask_of,
                            oracle_model, parts_of_mask, robot_scene_dicts, trace_inputs)


def edges_to_arrays(edges, n):
    base = np.array([e[0] for e in edges], dtype=np.int64).reshape(len(edges), n)
    mask = np.array([mask_of(e[1][0]) for e in edges], dtype=np.int64)
    return base, mask


def oracle_field(g, tag):
    if tag.startswith("kclf"):
        gbb = g[f"{tag}_gbb"]
        bar = g[f"{tag}_barrier"]
        n = g[f"{tag}_support"].shape[1]
        return O.Field.rbf(g[f"{tag}_support"], g[f"{tag}_weights"], gbb[0], gbb[1],
                           barrier=(bar[0], bar[1], bar[2:2 + n], bar[2 + n:]))
    kind, args = analytic_spec(tag)
    return getattr(O.Field, kind)(*args)


def run_oracle_trace(g, tag):
    inp = trace_inputs(g, tag)
    t = O.Trace(oracle_field(g, tag), inp["n"], inp["scale"], inp["offset"], inp["box"], inp["max_edges"], inp["eps"])
    return t.run(inp["seeds"]), inp


# ---- lattice -----------------------------------------------------------------------------------
@pytest.mark.parametrize("n", [2, 3, 4, 5, 6])
def test_expansion_plans_match_reference(golden, n):
    rows = golden("lattice")[f"plan_n{n}"]
    at = 0
    for mask in range(1, 1 << n):
        plan = O.expansion_plan(parts_of_mask(mask, n), n)
        for j, (c, bc, ac) in enumerate(plan):
            want = rows[at]
            got = [mask, j, *c, *bc[0], mask_of(bc[1][0]), int(bc[2]), *ac[0], mask_of(ac[1][0]), int(ac[2])]
            assert list(want) == got
            at += 1
    assert at == rows.shape[0]


@pytest.mark.parametrize("n", [2, 3, 4, 5, 6])
def test_cellcofaces_match_reference(golden, n):
    rows = golden("lattice")[f"cellcofaces_n{n}"]
    masks = list(dict.fromkeys(int(m) for m in rows[:, 0]))
    at = 0
    for mask in masks:
        cells = O.cellcofaces_of_edge(((0,) * n, parts_of_mask(mask, n)))
        for cell in cells:
            want = rows[at]
            assert list(want) == [mask, *cell[0], *[p[0] for p in cell[1][:-1]]]
            at += 1
    assert at == rows.shape[0]


def test_fig2_cell_edges(golden):
    g = golden("lattice")
    edges = O.pair_edges(((0, 0, 0), ((2,), (0,), (1,), (3,))))
    base, mask = edges_to_arrays(edges, 3)
    assert np.array_equal(base, g["fig2_cell_edges_base"])
    assert np.array_equal(mask, g["fig2_cell_edges_mask"])


@pytest.mark.parametrize("n", [2, 3, 5])
def test_locate_point(golden, n):
    g = golden("lattice")
    offset = tuple(0.05 * (i + 1) for i in range(n))
    for p, b, perm in zip(g[f"locate_n{n}_points"], g[f"locate_n{n}_base"], g[f"locate_n{n}_perm"]):
        cell = O.locate_point(p, 0.37, offset)
        assert list(cell[0]) == list(b)
        assert [q[0] for q in cell[1][:-1]] == list(perm)


# ---- traces ------------------------------------------------------------------------------------
@pytest.mark.parametrize("tag", ANALYTIC_TRACES + LEARNED_TRACES[:3])
def test_trace_matches_reference(golden, tag):
    g = golden("traces")
    t, inp = run_oracle_trace(g, tag)
    base, mask = edges_to_arrays(t.edges, inp["n"])
    assert np.array_equal(base, g[f"{tag}_edge_base"])          # same set AND admission order
    assert np.array_equal(mask, g[f"{tag}_edge_mask"])
    st = g[f"{tag}_stats"]
    assert [t.levels, t.seeds, len(t.visited), t.field_evaluations, t.dropped, int(t.complete), int(t.closure_ok)] == list(st[:7])
    stages = np.array([[("locate_cells", "cell_edges", "edge_cofaces", "coface_partner").index(s[0]), *s[1:]]
                       for s in t.stages])
    assert np.array_equal(stages, g[f"{tag}_stages"])
    if f"{tag}_adjacency" in g:
        assert np.array_equal(np.asarray(t.sorted_adjacency()).reshape(-1, 2), g[f"{tag}_adjacency"])
    pts = t.points()
    want = g[f"{tag}_points"]
    if tag.startswith("kclf"):
        assert np.allclose(pts, want, rtol=0, atol=1e-8)
    else:
        assert np.array_equal(pts, want)


def test_trace_n6_learned(golden):
    """6-D learned manifold: 35 728 edges; the oracle needs ~1 min, so only the set and flags."""
    g = golden("traces")
    t, inp = run_oracle_trace(g, "kclf_n6")
    base, mask = edges_to_arrays(t.edges, 6)
    assert np.array_equal(base, g["kclf_n6_edge_base"])
    assert np.array_equal(mask, g["kclf_n6_edge_mask"])
    assert [t.levels, t.field_evaluations, t.dropped, int(t.closure_ok)] == [int(g["kclf_n6_stats"][i]) for i in (0, 3, 4, 6)]
    adj = np.asarray(t.sorted_adjacency(), dtype=np.int64)
    digest = [adj.shape[0], int(adj[:, 0].sum()), int(adj[:, 1].sum()), int((adj[:, 0] * 31 + adj[:, 1]).sum() % (1 << 61))]
    assert digest == list(g["kclf_n6_adjacency_digest"])


@pytest.mark.parametrize("tag", LEARNED_TRACES)
def test_field_values(golden, tag):
    g = golden("traces")
    f = oracle_field(g, tag)
    got = f.values(g[f"{tag}_probe_points"])
    want = g[f"{tag}_probe_values"]
    tol = 1e-12 * (np.abs(g[f"{tag}_weights"]).sum() + abs(g[f"{tag}_gbb"][1]))
    assert np.max(np.abs(got - want)) <= tol


# ---- coarse cells + refine ----------------------------------------------------------------------
@pytest.mark.parametrize("tag", ["kclf_n3", "kclf_n4"])
def test_coarse_cells(golden, tag):
    g = golden("traces")
    n = g[f"{tag}_edge_base"].shape[1]
    edges = [(tuple(int(v) for v in b), parts_of_mask(int(m), n)) for b, m in zip(g[f"{tag}_edge_base"], g[f"{tag}_edge_mask"])]
    cells = O.coarse_cells(edges)
    base = np.array([c[0] for c in cells])
    perm = np.array([[p[0] for p in c[1][:-1]] for c in cells])
    assert np.array_equal(base, g[f"{tag}_cells_base"])
    assert np.array_equal(perm, g[f"{tag}_cells_perm"])


@pytest.mark.parametrize("n,k", [(2, 2), (3, 3), (5, 2), (6, 2), (4, 4)])
def test_template(golden, n, k):
    g = golden("refine")
    v, e, w = O.build_template(n, k)
    assert np.array_equal(v, g[f"template_n{n}_k{k}_v"])
    assert np.array_equal(e, g[f"template_n{n}_k{k}_e"])


@pytest.mark.parametrize("tag", ["sphere_n2_k3", "sphere_n3_k2", "sphere_n4_k2"])
def test_refine_analytic(golden, tag):
    g = golden("refine")
    n, lam, k = g[f"{tag}_params"]
    n, k = int(n), int(k)
    cells = [(tuple(int(v) for v in b), tuple((int(p),) for p in perm) + ((n,),))
             for b, perm in zip(g[f"{tag}_cells_base"], g[f"{tag}_cells_perm"])]
    out = O.refine(cells, O.build_template(n, k), O.Field.sphere(np.zeros(n), 0.8), lambda p: p[:, 0] > 0.1,
                   lam * k, np.zeros(n), k, 1e-9)
    assert np.array_equal(out["points"], g[f"{tag}_points"])
    assert np.array_equal(out["in_collision"], g[f"{tag}_labels"])
    assert sum(out["crossing_edges"]) == int(g[f"{tag}_crossings"][0])


def test_refine_learned_with_collision(golden):
    g = golden("traces")
    tag, n = "kclf_n3", 3
    cells = [(tuple(int(v) for v in b), tuple((int(p),) for p in perm) + ((n,),))
             for b, perm in zip(g[f"{tag}_cells_base"], g[f"{tag}_cells_perm"])]
    robot, scene = oracle_model(*robot_scene_dicts(n, 3))
    lat = g[f"{tag}_lattice"]
    out = O.refine(cells, O.build_template(n, 2), oracle_field(g, tag), lambda p: O.not_free(robot, scene, p),
                   float(lat[1]), lat[2:2 + n], 2, 1e-9, batch_cells=40)
    want = g[f"{tag}_refine_points"]
    assert out["points"].shape == want.shape
    assert np.allclose(out["points"], want, rtol=0, atol=1e-8)
    assert np.array_equal(out["in_collision"], g[f"{tag}_refine_labels"])
    rows = g[f"{tag}_refine_batches"]
    assert out["crossing_edges"] == list(rows[:, 2])
    assert out["new_points"] == list(rows[:, 3])


# ---- refine at n = 5 / 6: the oracle against the REAL reference's refine of cell subsets ---------------
def cells_sha(cb, cp):
    import hashlib
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(cb, dtype=np.int16).tobytes())
    h.update(np.ascontiguousarray(cp, dtype=np.uint8).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("tag", ["kclf_n5", "kclf_n6"])
def test_refine_high_dim_subsets(golden, tag):
    """subdivision.py:220-301 at the benchmarked dimensions: per-cell crossing counts, per-cell fresh points (the
    greedy eps-dedup over 3^n neighbour buckets, order-dependent), kept points and collision labels of the first /
    middle / last runs of sorted coarse cells, exactly as the reference produced them (one cell per batch)."""
    g, gh = golden("traces"), golden("refine_hd")
    n = g[f"{tag}_support"].shape[1]
    cells = [(tuple(int(v) for v in b), tuple((int(p),) for p in perm) + ((n,),))
             for b, perm in zip(gh[f"{tag}_sub_base"], gh[f"{tag}_sub_perm"])]
    robot, scene = oracle_model(*robot_scene_dicts(n, 8))
    lat = g[f"{tag}_lattice"]
    out = O.refine(cells, O.build_template(n, 2), oracle_field(g, tag), lambda p: O.not_free(robot, scene, p),
                   float(lat[1]), lat[2:2 + n], 2, 1e-9, batch_cells=1)
    rows = gh[f"{tag}_sub_per_cell"]
    assert out["crossing_edges"] == list(rows[:, 0])
    assert out["new_points"] == list(rows[:, 1])
    want = gh[f"{tag}_sub_points"]
    assert out["points"].shape == want.shape
    assert np.allclose(out["points"], want, rtol=0, atol=1e-8)
    assert np.array_equal(out["in_collision"], gh[f"{tag}_sub_labels"])
    assert out["eps_dedup"] == float(gh[f"{tag}_sub_eps_dedup"][0])


@pytest.mark.parametrize("tag", ["kclf_n5", "kclf_n6"])
def test_coarse_cells_high_dim_head(golden, tag):
    """coarse_cells (subdivision.py:132-141) of the first 3000 traced edges at n = 5 / 6: sha256 of the sorted list."""
    g, gh = golden("traces"), golden("refine_hd")
    n = g[f"{tag}_edge_base"].shape[1]
    edges = [(tuple(int(v) for v in b), parts_of_mask(int(m), n))
             for b, m in zip(g[f"{tag}_edge_base"][:3000], g[f"{tag}_edge_mask"][:3000])]
    cells = O.coarse_cells(edges)
    assert len(cells) == int(gh[f"{tag}_cells_head3000"][0])
    base = np.array([c[0] for c in cells])
    perm = np.array([[p[0] for p in c[1][:-1]] for c in cells])
    assert cells_sha(base, perm) == str(gh[f"{tag}_cells_head3000_sha256"][0])


# ---- collision -----------------------------------------------------------------------------------
@pytest.mark.parametrize("n,nobs", [(3, 3), (4, 3), (5, 8), (6, 8)])
def test_collision(golden, n, nobs):
    g = golden("collision")
    robot, scene = oracle_model(*robot_scene_dicts(n, nobs))
    q = g[f"coll_n{n}_q"]
    assert np.array_equal(O.not_free(robot, scene, q), g[f"coll_n{n}_unfree"])
    inside = np.all(np.abs(q) <= 1.5, axis=1)
    assert np.array_equal(O.batch_hits(robot, scene, q[inside]), g[f"coll_n{n}_hits_inside"])
    assert np.array_equal(O.fk_batch(robot, q[:40]), g[f"coll_n{n}_fk"])


def test_collision_prismatic_posed(golden):
    g = golden("collision")
    robot, scene = oracle_model(PRISM_ROBOT, PRISM_SCENE)
    q = g["coll_prism_q"]
    assert np.array_equal(O.batch_hits(robot, scene, q), g["coll_prism_hits"])
    assert np.allclose(O.fk_batch(robot, q[:40]), g["coll_prism_fk"], rtol=0, atol=1e-15)


# ---- backend seam ------------------------------------------------------------------------------------
def test_backend_kernels(golden):
    g = golden("backend")
    gamma, bias = g["rbf_params"]
    got = O.rbf_values(g["rbf_points"], g["rbf_support"], g["rbf_weights"], gamma, bias)
    assert np.array_equal(got, g["rbf_values"])      # same loop order as the Cython kernel
    c, r = g["hits_centers"], g["hits_radii"]
    assert np.array_equal(O.sphere_box_hits(c, r, 0.8, 0.5, 1.1), g["hits_box"])
    assert np.array_equal(O.sphere_cylinder_hits(c, r, 0.9, 0.4), g["hits_cyl"])
    assert np.array_equal(O.sphere_sphere_hits(c, r, 0.6), g["hits_sph"])
    tc, tr = g["touch_centers"], g["touch_radii"]
    assert np.array_equal(O.sphere_box_hits(tc, tr, 2.0, 2.0, 2.0), g["touch_box"])
    assert list(g["touch_box"]) == [1, 0, 0, 1, 0]    # pkg/tests/test_backends.py:52-69
    assert np.array_equal(O.sphere_cylinder_hits(tc, tr, 2.0, 1.0), g["touch_cyl"])
    assert np.array_equal(O.sphere_sphere_hits(tc, tr, 1.0), g["touch_sph"])


def test_rbf_multithreaded_is_identical(golden):
    g = golden("backend")
    gamma, bias = g["rbf_params"]
    O.THREADS = 4
    try:
        got = O.rbf_values(g["rbf_points"], g["rbf_support"], g["rbf_weights"], gamma, bias)
    finally:
        O.THREADS = 1
    assert np.array_equal(got, g["rbf_values"])


def test_bisection(golden):
    g = golden("backend")
    got = O.intersection_points_batch(O.Field.sphere(np.zeros(3), 1.0), g["bisect_a"], g["bisect_b"], 1e-9)
    assert np.array_equal(got, g["bisect_points"])
