"""Generate tests/golden/*.npz by running the REAL reference (permatrace) in this container.

    python tests/golden/make_golden.py            # needs /root/reference (read-only mount)

The reference cannot travel to the GPU box, so its outputs are frozen here as small fixtures; the
oracle (oracle/permatrace_oracle.py) and the CUDA path are both tested against them.  The Cython
backend is used when a scratch build exists (copy /root/reference/pkg to /tmp/refbuild and run
`python setup.py build_ext --inplace` there); otherwise the reference's numpy backend.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
for cand in ("/tmp/refbuild/pkg/src", "/root/reference/pkg/src"):
    if Path(cand, "permatrace").exists():
        sys.path.insert(0, cand)
        break
sys.path.insert(0, str(REPO))

import permatrace  # noqa: E402
from permatrace import lattice as rl  # noqa: E402
from permatrace import tracer as rt  # noqa: E402
from permatrace import manifold as rm  # noqa: E402
from permatrace import subdivision as rs  # noqa: E402
from permatrace import collision as rc  # noqa: E402
from permatrace import backend as rb  # noqa: E402
from permatrace.pipeline import Problem, _not_free_checker  # noqa: E402


def mask_of(part):
    m = 0
    for label in part:
        m |= 1 << label
    return m


def edge_arrays(edges, n):
    base = np.array([e.base for e in edges], dtype=np.int32).reshape(len(edges), n)
    mask = np.array([mask_of(e.parts[0]) for e in edges], dtype=np.uint32)
    return base, mask


def cell_arrays(cells, n):
    base = np.array([c.base for c in cells], dtype=np.int32).reshape(len(cells), n)
    perm = np.array([[p[0] for p in c.parts[:-1]] for c in cells], dtype=np.uint8).reshape(len(cells), n)
    return base, perm


def parts_of_mask(mask, n):
    p1 = tuple(d for d in range(n) if mask >> d & 1)
    p2 = tuple(d for d in range(n) if not mask >> d & 1) + (n,)
    return (p1, p2)


# ---- lattice -----------------------------------------------------------------------------------
def lattice_golden(out):
    for n in range(2, 7):
        rows = []
        for mask in range(1, 1 << n):
            parts = parts_of_mask(mask, n)
            plan = rt._expansion_plan(parts, n)
            for j, (c, bc, ac) in enumerate(plan):
                rows.append([mask, j, *c,
                             *bc[0], mask_of(bc[1][0]), int(bc[2]),
                             *ac[0], mask_of(ac[1][0]), int(ac[2])])
                # canonical partner edges always keep the wrap label in the second part
                assert n in bc[1][1] and n in ac[1][1]
        out[f"plan_n{n}"] = np.asarray(rows, dtype=np.int32)
    for n in range(2, 7):
        rows = []
        masks = range(1, 1 << n) if n <= 5 else [1, 3, 7, 15, 31, 63, 0b101010, 0b100000]
        for mask in masks:
            edge = rl.PermSimplex((0,) * n, parts_of_mask(mask, n))
            for cell in rl.cellcofaces_of_edge(edge):
                assert cell.parts[-1] == (n,)
                rows.append([mask, *cell.base, *[p[0] for p in cell.parts[:-1]]])
        out[f"cellcofaces_n{n}"] = np.asarray(rows, dtype=np.int16)
    # Fig. 2 worked example of the reference's own tests (test_lattice.py:64-93): cell edges order
    cell = rl.PermSimplex((0, 0, 0), ((2,), (0,), (1,), (3,)))
    b, m = edge_arrays(rl.edges_of_cell(cell), 3)
    out["fig2_cell_edges_base"], out["fig2_cell_edges_mask"] = b, m
    # locate_point on a 3^n block of perturbed points
    rng = np.random.default_rng(3)
    for n in (2, 3, 5):
        cfg = rl.LatticeConfig(n, 0.37, tuple(0.05 * (i + 1) for i in range(n)))
        pts = rng.uniform(-2, 2, size=(64, n))
        pts[:8] = np.round(pts[:8] / 0.37) * 0.37 + np.asarray(cfg.offset)   # on-lattice ties
        cells = [rl.locate_point(p, cfg) for p in pts]
        cb, cp = cell_arrays(cells, n)
        out[f"locate_n{n}_points"], out[f"locate_n{n}_base"], out[f"locate_n{n}_perm"] = pts, cb, cp


# ---- manifolds used by several sections ------------------------------------------------------------
def learned_manifold(n, S, lam, r_split, seed=0, limit=1.5):
    """SURVEY.md Appendix B recipe (mirrors pipeline.py:329-362)."""
    rng = np.random.default_rng(seed)
    x = rng.uniform(-limit, limit, size=(S, n))
    inside = np.linalg.norm(x, axis=1) < r_split
    gamma = 2.0
    sigma = 1.0 / np.sqrt(2.0 * gamma)
    lo, hi = -limit * np.ones(n), limit * np.ones(n)
    barrier = rm.BoxBarrier(lo, hi, scale=sigma / 4.0, gain=2.0 / sigma)
    m0 = rm.train_classifier(x[inside], x[~inside], gamma=gamma, regularization=1e-3, barrier=barrier)
    m = rm.KernelClassifierManifold(m0.support, m0.weights, m0.gamma, bias=m0.bias + lam * np.sqrt(2 * gamma),
                                    barrier=barrier)
    k = 2
    coarse = lam * k
    margin = max(3.0 * coarse, 2.0 * sigma + (1.0 + 2.0 * np.sqrt(n)) * coarse)
    cfg = rt.TraceConfig(rl.LatticeConfig(n, coarse), box=(tuple(lo - margin), tuple(hi + margin)))
    seeds = rm.sample_seeds(m, (lo, hi), 20, rng=rng, min_separation=coarse / 2.0)
    return m, cfg, seeds


def save_manifold(out, tag, m):
    out[f"{tag}_support"] = m.support
    out[f"{tag}_weights"] = m.weights
    out[f"{tag}_gbb"] = np.array([m.gamma, m.bias])
    bar = m.barrier
    out[f"{tag}_barrier"] = np.concatenate([[bar.scale, bar.gain], bar.lower, bar.upper])


def save_trace(out, tag, result, cfg, seeds, with_adjacency=True):
    n = cfg.lattice.dim
    b, m = edge_arrays(result.edges, n)
    out[f"{tag}_seeds"] = np.asarray(seeds, dtype=np.float64)
    out[f"{tag}_lattice"] = np.array([n, cfg.lattice.scale, *cfg.lattice.offset])
    if cfg.box is not None:
        out[f"{tag}_box"] = np.array([cfg.box[0], cfg.box[1]], dtype=np.float64)
    out[f"{tag}_cfg"] = np.array([cfg.max_edges, cfg.eps])
    out[f"{tag}_edge_base"], out[f"{tag}_edge_mask"] = b.astype(np.int16), m.astype(np.uint8)
    out[f"{tag}_points"] = result.points
    st = result.stats
    out[f"{tag}_stats"] = np.array([st.levels, st.seeds, st.visited_edges, st.field_evaluations,
                                    st.dropped_out_of_box, int(st.complete), int(st.closure_ok),
                                    -1 if st.polyline_closed is None else int(st.polyline_closed)], dtype=np.int64)
    out[f"{tag}_stages"] = np.array([[("locate_cells", "cell_edges", "edge_cofaces", "coface_partner").index(s.name),
                                      s.level, s.items, s.capacity, s.produced] for s in st.stages], dtype=np.int64)
    if with_adjacency:
        out[f"{tag}_adjacency"] = np.asarray(result.adjacency, dtype=np.int32).reshape(-1, 2)
    else:
        adj = np.asarray(result.adjacency, dtype=np.int64).reshape(-1, 2)
        out[f"{tag}_adjacency_digest"] = np.array([adj.shape[0], int(adj[:, 0].sum()), int(adj[:, 1].sum()),
                                                   int((adj[:, 0] * 31 + adj[:, 1]).sum() % (1 << 61))], dtype=np.int64)


# ---- traces ----------------------------------------------------------------------------------------
def trace_golden(out):
    # analytic spheres (acceptance test 02 shapes: r=0.8 centred, lambdas 0.5/0.25)
    for n, lam in ((2, 0.25), (3, 0.25), (4, 0.5), (5, 0.5)):
        f = rm.SphereManifold(np.zeros(n), 0.8)
        cfg = rt.TraceConfig(rl.LatticeConfig(n, lam))
        seeds = f.seed_point()[None, :]
        save_trace(out, f"sphere_n{n}", rt.trace(seeds, f, cfg), cfg, seeds)
    # off-centre ellipsoid with lattice offset and clamp box that drops edges
    f = rm.EllipsoidManifold([0.1, -0.2, 0.05], [0.9, 0.6, 0.7])
    cfg = rt.TraceConfig(rl.LatticeConfig(3, 0.2, (0.01, 0.02, 0.03)), box=((-0.5, -1, -1), (1.2, 1, 1)))
    seeds = f.seed_point()[None, :]
    res = rt.trace(seeds, f, cfg)
    assert res.stats.dropped_out_of_box > 0
    save_trace(out, "ellipsoid_box", res, cfg, seeds)
    # cap
    f = rm.SphereManifold(np.zeros(3), 0.8)
    cfg = rt.TraceConfig(rl.LatticeConfig(3, 0.2), max_edges=150)
    seeds = f.seed_point()[None, :]
    res = rt.trace(seeds, f, cfg)
    assert not res.stats.complete
    save_trace(out, "sphere_cap", res, cfg, seeds)
    # plane through several seeds
    f = rm.PlaneManifold([1.0, 0.5, -0.25], 0.1)
    cfg = rt.TraceConfig(rl.LatticeConfig(3, 0.5), box=((-1.5,) * 3, (1.5,) * 3))
    seeds = np.array([f.seed_point(), f.seed_point() + np.array([0.2, -0.4, 0.0])])
    seeds[1] -= (seeds[1] @ f.normal - f.offset) * f.normal / (f.normal @ f.normal)
    save_trace(out, "plane_box", rt.trace(seeds, f, cfg), cfg, seeds)
    # learned manifolds (Appendix B recipe)
    for tag, (n, S, lam, r) in {"kclf_n3": (3, 512, 0.2, 0.9), "kclf_n4": (4, 1024, 0.3, 0.9),
                                "kclf_n5": (5, 1024, 0.4, 0.9), "kclf_n6": (6, 1024, 0.45, 1.3)}.items():
        m, cfg, seeds = learned_manifold(n, S, lam, r)
        res = rt.trace(seeds, m, cfg)
        print(tag, "edges", len(res.edges), "levels", res.stats.levels, "evals", res.stats.field_evaluations,
              "closure", res.closure_ok)
        save_manifold(out, tag, m)
        save_trace(out, tag, res, cfg, seeds, with_adjacency=len(res.edges) < 5000)
        # field values / signs on probe points, and bisection on the traced edges' first rows
        rng = np.random.default_rng(11)
        probes = rng.uniform(-2.0, 2.0, size=(256, n))
        out[f"{tag}_probe_points"] = probes
        out[f"{tag}_probe_values"] = m.values(probes)
        if tag in ("kclf_n3", "kclf_n4"):
            cells = rs.coarse_cells(res)
            cb, cp = cell_arrays(cells, n)
            out[f"{tag}_cells_base"], out[f"{tag}_cells_perm"] = cb.astype(np.int16), cp
        else:
            cells = rs.coarse_cells(res) if n == 5 else None
            if cells is not None:
                out[f"{tag}_cells_count"] = np.array([len(cells)])
                cb, cp = cell_arrays(cells, n)
                out[f"{tag}_cells_digest"] = np.array([int(cb.sum()), int((cp.astype(np.int64) * np.arange(1, n + 1)).sum())])
        if tag == "kclf_n3":
            refine_golden(out, tag, m, cfg, cells, n)


# ---- refine ------------------------------------------------------------------------------------------
def robot_scene(n, n_obstacles, seed=7):
    from paper_2406_04795_b200.scenes import arm_robot_dict, arm_scene_dict
    robot = rc.robot_from_dict(arm_robot_dict(n))
    scene = rc.scene_from_dict(arm_scene_dict(n_obstacles, seed))
    return robot, scene


class _Prob:
    def __init__(self, robot, scene):
        self.robot, self.scene = robot, scene

    def limits(self):
        return rc.joint_limits(self.robot)


def refine_golden(out, tag, m, cfg, cells, n):
    robot, scene = robot_scene(n, 3)
    checker = _not_free_checker(_Prob(robot, scene))
    template = rs.build_template(n, 2)
    res = rs.refine(cells, template, m, checker, cfg, memory_budget=None)
    res2 = rs.refine(cells, template, m, checker, cfg, memory_budget=40 * rs._cell_bytes(template))
    assert np.array_equal(res.points, res2.points)
    print(tag, "refine points", res.points.shape, "free", res.free_points.shape[0],
          "crossings", sum(b.crossing_edges for b in res.batch_stats))
    out[f"{tag}_refine_points"] = res.points
    out[f"{tag}_refine_labels"] = res.in_collision
    out[f"{tag}_refine_eps_dedup"] = np.array([res.eps_dedup])
    out[f"{tag}_refine_batches"] = np.array([[b.cells, b.fine_vertices, b.crossing_edges, b.new_points]
                                             for b in res2.batch_stats], dtype=np.int64)
    out[f"{tag}_refine_budget"] = np.array([40 * rs._cell_bytes(template)])


def refine_analytic_golden(out):
    for tag, n, lam, k in (("sphere_n2_k3", 2, 0.3, 3), ("sphere_n3_k2", 3, 0.4, 2), ("sphere_n4_k2", 4, 0.5, 2)):
        f = rm.SphereManifold(np.zeros(n), 0.8)
        cfg = rt.TraceConfig(rl.LatticeConfig(n, lam * k))
        res = rt.trace(f.seed_point()[None, :], f, cfg)
        cells = rs.coarse_cells(res)
        template = rs.build_template(n, k)
        ref = rs.refine(cells, template, f, lambda p: p[:, 0] > 0.1, cfg)
        print(tag, "cells", len(cells), "points", ref.points.shape[0])
        out[f"{tag}_params"] = np.array([n, lam, k])
        cb, cp = cell_arrays(cells, n)
        out[f"{tag}_cells_base"], out[f"{tag}_cells_perm"] = cb.astype(np.int16), cp
        out[f"{tag}_points"] = ref.points
        out[f"{tag}_labels"] = ref.in_collision
        out[f"{tag}_crossings"] = np.array([sum(b.crossing_edges for b in ref.batch_stats)])
        out[f"{tag}_template_v"] = template.vertices
        out[f"{tag}_template_e"] = template.edges
    for n, k in ((2, 2), (3, 3), (5, 2), (6, 2), (4, 4)):
        t = rs.build_template(n, k)
        out[f"template_n{n}_k{k}_v"] = t.vertices.astype(np.int8)
        out[f"template_n{n}_k{k}_e"] = t.edges.astype(np.int16)


# ---- refine at n = 5 / 6 (the benchmarked dimension): REAL reference on cell subsets --------------------
def cells_sha(cb, cp):
    """Digest of a sorted cell list: sha256 over the int16 bases followed by the uint8 permutations."""
    import hashlib
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(cb, dtype=np.int16).tobytes())
    h.update(np.ascontiguousarray(cp, dtype=np.uint8).tobytes())
    return h.hexdigest()


def refine_hd_golden(out):
    """subdivision.refine of the real reference (eps-dedup with its 3^n neighbour scan and the collision labels
    included) on three contiguous runs -- first / middle / last -- of the sorted coarse cells of the n = 5 and n = 6
    learned traces, ONE CELL PER BATCH so that per-cell crossing counts and per-cell fresh-point counts are pinned
    too; plus the digest of the FULL n = 6 coarse_cells list."""
    for tag, (n, S, lam, r, nobs, run) in {"kclf_n5": (5, 1024, 0.4, 0.9, 8, 130),
                                           "kclf_n6": (6, 1024, 0.45, 1.3, 8, 110)}.items():
        m, cfg, seeds = learned_manifold(n, S, lam, r)
        res = rt.trace(seeds, m, cfg)
        cells = rs.coarse_cells(res)
        cb, cp = cell_arrays(cells, n)
        out[f"{tag}_cells_count"] = np.array([len(cells)])
        out[f"{tag}_cells_sha256"] = np.array([cells_sha(cb, cp)])
        out[f"{tag}_cells_digest"] = np.array([int(cb.sum()), int((cp.astype(np.int64) * np.arange(1, n + 1)).sum())])
        # cells of the first 3000 traced edges only: small enough for the pure-Python oracle in the CPU suite
        head = rs.coarse_cells(SimpleNamespace(edges=res.edges[:3000]))
        hb, hp = cell_arrays(head, n)
        out[f"{tag}_cells_head3000"] = np.array([len(head)])
        out[f"{tag}_cells_head3000_sha256"] = np.array([cells_sha(hb, hp)])
        mid = len(cells) // 2
        pick = list(range(run)) + list(range(mid - run // 2, mid - run // 2 + run)) + list(range(len(cells) - run, len(cells)))
        subset = [cells[i] for i in pick]
        robot, scene = robot_scene(n, nobs)
        checker = _not_free_checker(_Prob(robot, scene))
        template = rs.build_template(n, 2)
        ref = rs.refine(subset, template, m, checker, cfg, memory_budget=rs._cell_bytes(template))
        whole = rs.refine(subset, template, m, checker, cfg)
        assert np.array_equal(ref.points, whole.points) and np.array_equal(ref.in_collision, whole.in_collision)
        assert len(ref.batch_stats) == len(subset)
        print(tag, "cells", len(cells), "subset", len(subset), "crossings", sum(b.crossing_edges for b in ref.batch_stats),
              "points", ref.points.shape[0], "free", ref.free_points.shape[0])
        out[f"{tag}_pick"] = np.asarray(pick, dtype=np.int64)
        sb, sp = cell_arrays(subset, n)
        out[f"{tag}_sub_base"], out[f"{tag}_sub_perm"] = sb.astype(np.int16), sp
        out[f"{tag}_sub_per_cell"] = np.array([[b.crossing_edges, b.new_points] for b in ref.batch_stats], dtype=np.int32)
        out[f"{tag}_sub_points"] = ref.points
        out[f"{tag}_sub_labels"] = ref.in_collision
        out[f"{tag}_sub_eps_dedup"] = np.array([ref.eps_dedup])


# ---- collision -----------------------------------------------------------------------------------------
def collision_golden(out):
    rng = np.random.default_rng(5)
    for n, nobs in ((3, 3), (4, 3), (5, 8), (6, 8)):
        robot, scene = robot_scene(n, nobs)
        q = rng.uniform(-1.7, 1.7, size=(1500, n))          # some rows violate the +-1.5 limits
        inside = np.all(np.abs(q) <= 1.5, axis=1)
        out[f"coll_n{n}_q"] = q
        out[f"coll_n{n}_unfree"] = rc.batch_check(q, robot, scene, on_limit="unfree")
        out[f"coll_n{n}_hits_inside"] = rc._batch_hits(robot, scene, q[inside])
        out[f"coll_n{n}_fk"] = rc.fk_batch(robot, q[:40])
    # prismatic joint + posed obstacles
    robot = rc.robot_from_dict({
        "joints": [
            {"type": "prismatic", "axis": [1, 0, 0], "origin": {"xyz": [0, 0, 0.1], "rpy": [0.1, 0.2, 0.3]}, "limits": [-1, 1]},
            {"type": "revolute", "axis": [0, 1, 1], "origin": {"xyz": [0.3, 0, 0], "rpy": [0, 0, 0]}, "limits": [-2, 2]},
        ],
        "spheres": [{"link": 0, "offset": [0, 0, 0], "radius": 0.1}, {"link": 2, "offset": [0.2, 0.1, 0], "radius": 0.05},
                    {"link": 1, "offset": [0.1, 0, 0], "radius": 0.07}],
    })
    scene = rc.scene_from_dict({"obstacles": [
        {"type": "cylinder", "height": 0.5, "radius": 0.2, "origin": {"xyz": [0.6, 0.1, 0.0], "rpy": [0.5, 0.1, 0.0]}},
        {"type": "sphere", "radius": 0.25, "origin": {"xyz": [-0.7, 0.0, 0.2]}},
        {"type": "box", "size": [0.3, 0.2, 0.4], "origin": {"xyz": [0.1, 0.6, 0.0], "rpy": [0, 0, 0.7]}}]})
    q = rng.uniform([-1, -2], [1, 2], size=(800, 2))
    out["coll_prism_q"] = q
    out["coll_prism_hits"] = rc.batch_check(q, robot, scene)
    out["coll_prism_fk"] = rc.fk_batch(robot, q[:40])


# ---- backend seam -----------------------------------------------------------------------------------------
def backend_golden(out):
    rng = np.random.default_rng(9)
    pts, sup, w = rng.normal(size=(300, 4)), rng.normal(size=(150, 4)), rng.normal(size=150)
    out["rbf_points"], out["rbf_support"], out["rbf_weights"] = pts, sup, w
    out["rbf_params"] = np.array([0.7, -0.3])
    out["rbf_values"] = rb.rbf_values(pts, sup, w, 0.7, -0.3)
    c = rng.uniform(-1.2, 1.2, size=(4000, 3))
    r = rng.uniform(0.01, 0.5, size=4000)
    out["hits_centers"], out["hits_radii"] = c, r
    out["hits_box"] = rb.sphere_box_hits(c, r, 0.8, 0.5, 1.1)
    out["hits_cyl"] = rb.sphere_cylinder_hits(c, r, 0.9, 0.4)
    out["hits_sph"] = rb.sphere_sphere_hits(c, r, 0.6)
    # exact-touch dyadic cases of the reference's own test (pkg/tests/test_backends.py:52-69)
    centers = np.array([[1.5, 0.0, 0.0], [1.5 + 2.0 ** -20, 0.0, 0.0], [2.0, 2.0, 0.0], [1.0, 1.0, 1.0], [1.75, 1.75, 1.75]])
    radii = np.array([0.5, 0.5, 0.5, 0.25, 1.0])
    out["touch_centers"], out["touch_radii"] = centers, radii
    out["touch_box"] = rb.sphere_box_hits(centers, radii, 2.0, 2.0, 2.0)
    out["touch_cyl"] = rb.sphere_cylinder_hits(centers, radii, 2.0, 1.0)
    out["touch_sph"] = rb.sphere_sphere_hits(centers, radii, 1.0)
    # bisection on an analytic field
    f = rm.SphereManifold(np.zeros(3), 1.0)
    a = rng.uniform(-0.5, 0.5, size=(200, 3))
    b = a + rng.normal(size=(200, 3))
    b *= (1.2 + rng.uniform(size=(200, 1))) / np.linalg.norm(b, axis=1, keepdims=True)
    out["bisect_a"], out["bisect_b"] = a, b
    out["bisect_points"] = rm.intersection_points_batch(f, a, b, 1e-9)


def proof_golden(out):
    """The reference's own solve() on its bundled wall2d scene -> an infeasibility certificate, and the
    reference's verify_proof() verdicts on the intact certificate and on a tamper matrix."""
    import copy
    import json
    from permatrace import pipeline as pl
    scene_path = Path(pl.__file__).parent / "scenes" / "wall2d.yaml"
    pf = pl.load_problem_file(scene_path)
    problem = pf.problem(None, None)
    proof = pl.solve(problem, pl.SolveParams(lam=0.04, k=2, gamma=60.0))
    assert isinstance(proof, pl.InfeasibilityProof)
    m = proof.manifold
    out["robot_scene_json"] = np.array([json.dumps({"robot": pl.robot_to_dict(problem.robot), "scene": pl.scene_to_dict(problem.scene)})])
    out["start"], out["goal"] = problem.q_start, problem.q_goal
    out["support"], out["weights"] = m.support, m.weights
    out["gbb"] = np.array([m.gamma, m.bias])
    b = m.barrier
    out["barrier"] = np.concatenate([[b.scale, b.gain], b.lower, b.upper])
    out["params"] = np.array([proof.lam, proof.k, proof.eps, proof.f_start, proof.f_goal, proof.coarse_edges, proof.coarse_cells,
                              float(proof.closure_ok), -1.0 if proof.polyline_closed is None else float(proof.polyline_closed)])
    out["points"] = proof.points
    out["fingerprint"] = np.array([proof.fingerprint])

    def tampered(kind):
        p = copy.copy(proof)
        if kind == "fingerprint":
            p.fingerprint = "0" * 64
        elif kind == "point_moved":
            p.points = proof.points.copy(); p.points[3, 0] += 1e-3
        elif kind == "point_dropped":
            p.points = proof.points[1:].copy()
        elif kind == "f_start":
            p.f_start = proof.f_start + 1e-3
        elif kind == "closure_flag":
            p.closure_ok = False
        elif kind == "coarse_edges":
            p.coarse_edges = proof.coarse_edges + 1
        elif kind == "coarse_cells":
            p.coarse_cells = proof.coarse_cells - 1
        elif kind == "bias_shift":
            p.manifold = pl.KernelClassifierManifold(m.support, m.weights, m.gamma, m.bias + 0.05, barrier=m.barrier)
        elif kind == "point_free":
            p.points = proof.points.copy(); p.points[0] = problem.q_start
        return p

    kinds = ["intact", "fingerprint", "point_moved", "point_dropped", "f_start", "closure_flag", "coarse_edges", "coarse_cells",
             "bias_shift", "point_free"]
    names, verdicts = [], []
    for kind in kinds:
        rep = pl.verify_proof(tampered(kind), problem)
        names.append(json.dumps([c.name for c in rep.checks]))
        verdicts.append(json.dumps([bool(c.passed) for c in rep.checks]))
        print(f"  {kind:14s} ok={rep.ok} {[(c.name, c.passed) for c in rep.checks if not c.passed]}")
    out["tamper_kinds"] = np.array(kinds)
    out["tamper_check_names"] = np.array(names)
    out["tamper_check_passed"] = np.array(verdicts)


def solve_golden(out):
    """The reference's own solve() on its three bundled scenes (wall2d -> proof, gap2d -> plan, arm3wall -> proof):
    the per-iteration record of the loop (roadmap size, class sizes, trace/refine counts, skips), the roadmap the
    planner ended with, and the outcome (certificate points / plan path).  Pins `pipeline.solve` + `planner`."""
    import json
    import time
    from permatrace import pipeline as pl
    keys = ("iteration", "roadmap", "positive", "negative", "edges", "cells", "points", "free_points")
    for name in ("wall2d", "gap2d", "arm3wall"):
        pf = pl.load_problem_file(Path(pl.__file__).parent / "scenes" / f"{name}.yaml")
        problem = pf.problem(None, None)
        params = pf.solve_params(timeout=3600.0)
        captured = {}
        stats_cls, roadmap_cls = pl.SolveStats, pl.Roadmap

        def stats_factory():
            captured["stats"] = stats_cls()
            return captured["stats"]

        def roadmap_factory(*a, **kw):
            captured["roadmap"] = roadmap_cls(*a, **kw)
            return captured["roadmap"]

        pl.SolveStats, pl.Roadmap = stats_factory, roadmap_factory
        try:
            t0 = time.perf_counter()
            outcome = pl.solve(problem, params)
            dt = time.perf_counter() - t0
        finally:
            pl.SolveStats, pl.Roadmap = stats_cls, roadmap_cls
        rec = captured["stats"].iterations
        out[f"{name}/records"] = np.array([[float(r.get(k, -1)) for k in keys] for r in rec])
        out[f"{name}/skips"] = np.array([r.get("skip", "") for r in rec])
        rm_ = captured["roadmap"]
        out[f"{name}/roadmap_configs"] = np.asarray(rm_.configs)
        out[f"{name}/roadmap_free"] = np.asarray(rm_.free)
        out[f"{name}/roadmap_degree"] = np.array([len(d) for d in rm_.neighbors])
        out[f"{name}/robot_scene_json"] = np.array([json.dumps({"robot": pl.robot_to_dict(problem.robot), "scene": pl.scene_to_dict(problem.scene)})])
        out[f"{name}/start"], out[f"{name}/goal"] = problem.q_start, problem.q_goal
        out[f"{name}/params_json"] = np.array([json.dumps(pf.params)])
        out[f"{name}/seconds"] = np.array([dt])
        if isinstance(outcome, pl.InfeasibilityProof):
            m = outcome.manifold
            out[f"{name}/outcome"] = np.array(["proof"])
            out[f"{name}/support"], out[f"{name}/weights"] = m.support, m.weights
            out[f"{name}/gbb"] = np.array([m.gamma, m.bias])
            out[f"{name}/points"] = outcome.points
            out[f"{name}/counts"] = np.array([outcome.coarse_edges, outcome.coarse_cells, int(outcome.meta["iterations"])])
            out[f"{name}/f"] = np.array([outcome.f_start, outcome.f_goal])
            print(f"  {name}: proof after {outcome.meta['iterations']} iterations, {outcome.points.shape[0]} points, {dt:.1f} s")
        elif isinstance(outcome, pl.Plan):
            out[f"{name}/outcome"] = np.array(["plan"])
            out[f"{name}/path"] = np.asarray(outcome.path)
            print(f"  {name}: plan with {len(outcome.path)} waypoints after {len(rec)} iterations, {dt:.1f} s")
        else:
            raise AssertionError(f"{name}: unexpected outcome {outcome!r}")
    out["record_keys"] = np.array(keys)


def main():
    print("reference backend:", permatrace.BACKEND, "from", permatrace.__file__)
    sections = {"lattice": lattice_golden, "traces": trace_golden, "refine": refine_analytic_golden, "refine_hd": refine_hd_golden,
                "collision": collision_golden, "backend": backend_golden, "proof": proof_golden, "solve": solve_golden}
    only = sys.argv[1:] or list(sections)
    for name in only:
        out: dict = {"reference_backend": np.array([permatrace.BACKEND])}
        sections[name](out)
        path = HERE / f"{name}.npz"
        np.savez_compressed(path, **out)
        print(f"wrote {path} ({path.stat().st_size / 1024:.0f} KiB, {len(out)} arrays)")


if __name__ == "__main__":
    main()
