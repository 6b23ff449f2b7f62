"""The solve loop and its roadmap against the REAL reference.

tests/golden/solve.npz (tests/golden/make_golden.py::solve_golden) holds what the reference's own `solve()` did on its
three bundled scenes: wall2d -> infeasibility proof after 4 iterations, gap2d -> plan, arm3wall (3-DoF arm) -> proof
after 6 iterations / 227 s on the CPU; per-iteration records, the final roadmap and the outcome.

CPU tests pin the host logic (roadmap planning with batched collision verdicts, batched seed projection, random-stream
bookkeeping) with the oracle's collision predicate injected; the GPU tests run the product `solve()` end to end."""

from __future__ import annotations

import json

import numpy as np
import pytest

from tests.conftest import oracle_model

KEYS = ("iteration", "roadmap", "positive", "negative", "edges", "cells", "points", "free_points")


def _problem(g, name, cls=None):
    from paper_2406_04795_b200 import collision as CO
    rs = json.loads(str(g[f"{name}/robot_scene_json"][0]))
    robot, scene = CO.robot_from_dict(rs["robot"]), CO.scene_from_dict(rs["scene"])
    return robot, scene, rs


def _oracle_check(rs):
    from oracle import permatrace_oracle as O
    robot, scene = oracle_model(rs["robot"], rs["scene"])
    return lambda pts: O.batch_hits(robot, scene, np.ascontiguousarray(pts, dtype=np.float64))


# ---- host logic (no GPU) ----------------------------------------------------------------------------------
def test_roadmap_growth_matches_reference_roadmap(golden):
    """One `grow(500)` on gap2d, collision verdicts from the oracle in TWO batches: same vertices, same free flags,
    same degrees, same shortest path as the roadmap the reference built with one batch per vertex."""
    from paper_2406_04795_b200 import planner as PLN
    g = golden("solve")
    robot, scene, rs = _problem(g, "gap2d")
    rng = np.random.default_rng(0)
    roadmap = PLN.Roadmap(robot, scene, delta=0.04 / 4.0, knn=10, rng=rng, check=_oracle_check(rs))
    roadmap.add_config(g["gap2d/start"], free=True)
    roadmap.add_config(g["gap2d/goal"], free=True)
    free_added = PLN.grow(roadmap, 500)
    assert roadmap.collision_batches == 2
    assert np.array_equal(np.asarray(roadmap.configs), g["gap2d/roadmap_configs"])
    assert np.array_equal(np.asarray(roadmap.free), g["gap2d/roadmap_free"])
    assert free_added == int(g["gap2d/roadmap_free"].sum()) - 2
    assert np.array_equal(np.array([len(d) for d in roadmap.neighbors]), g["gap2d/roadmap_degree"])
    path = PLN.find_path(roadmap, g["gap2d/start"], g["gap2d/goal"])
    assert np.array_equal(np.asarray(path), g["gap2d/path"])
    assert roadmap.first_blocked_segment(path, roadmap.delta / 2.0) is None
    labels = PLN.labeled_samples(roadmap, g["gap2d/start"])
    assert len(labels.positive) + len(labels.negative) == len(roadmap)


def test_roadmap_first_iteration_prefix_on_proof_scenes(golden):
    """wall2d / arm3wall: the first grow() reproduces the first samples_per_iter+2 vertices of the reference's final
    roadmap, and the class sizes of its first iteration record."""
    from paper_2406_04795_b200 import planner as PLN
    g = golden("solve")
    for name, lam, count in (("wall2d", 0.04, 500), ("arm3wall", 0.15, 600)):
        robot, scene, rs = _problem(g, name)
        roadmap = PLN.Roadmap(robot, scene, delta=lam / 4.0, knn=10, rng=np.random.default_rng(0), check=_oracle_check(rs))
        roadmap.add_config(g[f"{name}/start"], free=True)
        roadmap.add_config(g[f"{name}/goal"], free=True)
        PLN.grow(roadmap, count)
        m = len(roadmap)
        assert m == count + 2 == int(g[f"{name}/records"][0][1])
        assert np.array_equal(np.asarray(roadmap.configs), g[f"{name}/roadmap_configs"][:m])
        assert np.array_equal(np.asarray(roadmap.free), g[f"{name}/roadmap_free"][:m])
        assert PLN.find_path(roadmap, g[f"{name}/start"], g[f"{name}/goal"]) is None
        labels = PLN.labeled_samples(roadmap, g[f"{name}/start"])
        assert (len(labels.positive), len(labels.negative)) == tuple(int(v) for v in g[f"{name}/records"][0][2:4])


def test_insert_free_points_equals_one_by_one(golden):
    """Batched insertion == the reference's sequential add_config + connect per point."""
    from paper_2406_04795_b200 import planner as PLN
    g = golden("solve")
    robot, scene, rs = _problem(g, "gap2d")
    check = _oracle_check(rs)
    maps = []
    for mode in ("batched", "sequential"):
        rm = PLN.Roadmap(robot, scene, delta=0.01, knn=6, rng=np.random.default_rng(3), check=check)
        PLN.grow(rm, 120)
        pts = np.random.default_rng(5).uniform(0.0, 1.0, (80, 2))
        pts = pts[~check(pts)]
        pts = np.vstack([pts, pts[:5] + 1e-4])           # near-duplicates are skipped
        if mode == "batched":
            before = rm.collision_batches
            added = PLN.insert_free_points(rm, pts, dedup_tol=1e-3)
            assert rm.collision_batches == before + 1
        else:
            added = 0
            for q in pts:
                if np.linalg.norm(np.asarray(rm.configs) - q, axis=1).min() <= 1e-3:
                    continue
                rm.connect(rm.add_config(q, free=True))
                added += 1
        maps.append((added, [dict(d) for d in rm.neighbors], np.asarray(rm.configs)))
    assert maps[0][0] == maps[1][0] == len(maps[0][2]) - 120
    assert maps[0][1] == maps[1][1] and np.array_equal(maps[0][2], maps[1][2])


class _NumpySphere:
    """Duck-typed manifold evaluated with numpy (host-logic tests only)."""

    dim = 3

    def values(self, pts):
        pts = np.atleast_2d(pts)
        return np.einsum("ij,ij->i", pts, pts) - 0.49 + 0.05 * np.sin(3.0 * pts[:, 0])

    def value(self, q):
        return float(self.values(q[None])[0])

    def gradient(self, q):
        g = 2.0 * np.asarray(q, dtype=np.float64)
        g[0] += 0.15 * np.cos(3.0 * q[0])
        return g


def test_batched_seed_projection_equals_sequential_loop():
    """sample_seeds: same seeds and the same generator state as the reference's draw-project-accept loop."""
    from paper_2406_04795_b200 import manifold as M
    m = _NumpySphere()
    box = (np.full(3, -1.0), np.full(3, 1.0))
    for count, sep in ((5, 0.0), (12, 0.3), (40, 0.5)):
        rng_a, rng_b = np.random.default_rng(11), np.random.default_rng(11)
        got = M.sample_seeds(m, box, count, rng=rng_a, min_separation=sep)
        kept, attempts = [], 0
        while len(kept) < count and attempts < 20 * count:
            attempts += 1
            start = rng_b.uniform(box[0], box[1])
            try:
                q = M.project_to_manifold(start, m)
            except M.ProjectionError:
                continue
            if sep > 0.0 and kept and np.min(np.linalg.norm(np.asarray(kept) - q, axis=1)) < sep:
                continue
            kept.append(q)
        assert np.array_equal(got, np.asarray(kept).reshape(len(kept), 3))
        assert rng_a.bit_generator.state == rng_b.bit_generator.state
        assert np.all(np.abs(m.values(got)) <= 1e-8)


def test_scene_file_parameters_and_errors(tmp_path, golden):
    from paper_2406_04795_b200 import pipeline as PL
    g = golden("solve")
    rs = json.loads(str(g["arm3wall/robot_scene_json"][0]))
    data = {"robot": rs["robot"], "scene": rs["scene"],
            "problem": {"start": g["arm3wall/start"].tolist(), "goal": g["arm3wall/goal"].tolist(),
                        "params": json.loads(str(g["arm3wall/params_json"][0]))}}
    import yaml
    path = tmp_path / "arm.yaml"
    path.write_text(yaml.safe_dump(data))
    pf = PL.load_problem_file(path)
    params = pf.solve_params(timeout=5.0)
    assert (params.lam, params.k, params.gamma, params.samples_per_iter, params.timeout) == (0.15, 2, 2.0, 600, 5.0)
    with pytest.raises(ValueError):
        pf.solve_params(nonsense=1)
    with pytest.raises(ValueError):
        PL.problem_file_from_dict({"robot": rs["robot"]})
    with pytest.raises(ValueError):
        PL.SolveParams(lam=0.0)
    pf.params["bogus"] = 1
    with pytest.raises(ValueError):
        pf.solve_params()
    no_endpoints = PL.problem_file_from_dict({"robot": rs["robot"], "scene": rs["scene"]})
    with pytest.raises(ValueError):
        no_endpoints.problem()


# ---- the product, end to end on the device ------------------------------------------------------------------
def _solve(g, name, **overrides):
    from paper_2406_04795_b200 import pipeline as PL
    robot, scene, _ = _problem(g, name)
    pf = PL.ProblemFile(robot, scene, g[f"{name}/start"], g[f"{name}/goal"], json.loads(str(g[f"{name}/params_json"][0])))
    problem = pf.problem()
    return problem, PL.solve(problem, pf.solve_params(timeout=600.0, **overrides))


def _records(stats):
    return np.array([[float(r.get(k, -1)) for k in KEYS] for r in stats.iterations])


@pytest.mark.gpu
def test_solve_gap2d_finds_the_reference_plan(golden):
    from paper_2406_04795_b200 import pipeline as PL
    g = golden("solve")
    _, outcome = _solve(g, "gap2d")
    assert isinstance(outcome, PL.Plan) and outcome.stats.outcome == "plan"
    assert np.array_equal(np.asarray(outcome.path), g["gap2d/path"])
    assert np.array_equal(_records(outcome.stats), g["gap2d/records"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["wall2d", "arm3wall"])
def test_solve_proves_infeasibility_like_the_reference(golden, name):
    """Same loop trajectory as the reference (iteration count, roadmap and class sizes, coarse edges, coarse cells,
    certificate points and free points of EVERY iteration), same final manifold within round-off, certificate points
    within 1e-5 relative, and the certificate verifies."""
    from paper_2406_04795_b200 import pipeline as PL
    g = golden("solve")
    problem, outcome = _solve(g, name)
    assert isinstance(outcome, PL.InfeasibilityProof)
    assert np.array_equal(_records(outcome.stats), g[f"{name}/records"])
    assert [r.get("skip", "") for r in outcome.stats.iterations] == [str(s) for s in g[f"{name}/skips"]]
    edges, cells, iters = (int(v) for v in g[f"{name}/counts"])
    assert (outcome.coarse_edges, outcome.coarse_cells, int(outcome.meta["iterations"])) == (edges, cells, iters)
    m = outcome.manifold
    # the support set contains the free certificate points fed back by earlier iterations (root-solve round-off)
    assert m.support.shape == g[f"{name}/support"].shape
    assert np.max(np.abs(m.support - g[f"{name}/support"])) <= 1e-7
    assert np.max(np.abs(m.weights - g[f"{name}/weights"])) <= 1e-4 * np.abs(g[f"{name}/weights"]).max()
    assert (m.gamma, m.bias) == tuple(g[f"{name}/gbb"])
    ref = g[f"{name}/points"]
    assert outcome.points.shape == ref.shape
    assert np.max(np.abs(outcome.points - ref)) <= 1e-5 * max(1.0, np.abs(ref).max())
    assert np.allclose([outcome.f_start, outcome.f_goal], g[f"{name}/f"], rtol=1e-9, atol=1e-12)
    assert PL.verify_proof(outcome, problem).ok


@pytest.mark.gpu
def test_solve_is_deterministic_and_records_stats(golden):
    """Reference test_pipeline.py:137-147: a rerun yields the same certificate, and every iteration leaves a record."""
    from paper_2406_04795_b200 import pipeline as PL
    g = golden("solve")
    _, a = _solve(g, "wall2d")
    _, b = _solve(g, "wall2d")
    assert isinstance(a, PL.InfeasibilityProof) and isinstance(b, PL.InfeasibilityProof)
    assert np.array_equal(a.points, b.points) and np.array_equal(a.manifold.weights, b.manifold.weights)
    assert (a.coarse_edges, a.coarse_cells, a.f_start, a.f_goal) == (b.coarse_edges, b.coarse_cells, b.f_start, b.f_goal)
    assert a.stats.outcome == "proof" and a.stats.seconds > 0.0
    assert len(a.stats.iterations) == int(a.meta["iterations"])
    last = a.stats.iterations[-1]
    assert {"roadmap", "positive", "negative", "train_s", "trace_s", "edges", "cells", "refine_s", "points", "free_points"} <= set(last)
    assert last["free_points"] == 0 and last["points"] == a.points.shape[0]


@pytest.mark.gpu
def test_solve_budgets(golden):
    """Reference test_pipeline.py:181-196: an expired clock and an exhausted iteration budget both end in SolveTimeout."""
    from paper_2406_04795_b200 import pipeline as PL
    g = golden("solve")
    _, outcome = _solve(g, "wall2d", max_iters=1)
    assert isinstance(outcome, PL.SolveTimeout) and outcome.reason == "iteration budget exhausted"
    assert outcome.stats.outcome == "timeout" and len(outcome.stats.iterations) == 1
    robot, scene, _ = _problem(g, "wall2d")
    pf = PL.ProblemFile(robot, scene, g["wall2d/start"], g["wall2d/goal"], json.loads(str(g["wall2d/params_json"][0])))
    outcome = PL.solve(pf.problem(), pf.solve_params(timeout=0.0))
    assert isinstance(outcome, PL.SolveTimeout) and outcome.reason == "wall-clock timeout"


@pytest.mark.gpu
def test_problem_rejects_bad_endpoints(golden):
    """Reference test_pipeline.py:50-62."""
    from paper_2406_04795_b200 import pipeline as PL
    g = golden("solve")
    robot, scene, _ = _problem(g, "wall2d")
    with pytest.raises(ValueError):
        PL.Problem(robot, scene, [0.5, 0.5], g["wall2d/goal"])            # inside the wall
    with pytest.raises(ValueError):
        PL.Problem(robot, scene, [1.5, 0.5], g["wall2d/goal"])            # outside the limits
    with pytest.raises(ValueError):
        PL.Problem(robot, scene, [0.15, 0.5, 0.0], g["wall2d/goal"])      # wrong width
    a, b = PL.Problem(robot, scene, g["wall2d/start"], g["wall2d/goal"]), None
    robot2, scene2, _ = _problem(g, "gap2d")
    b = PL.Problem(robot2, scene2, g["gap2d/start"], g["gap2d/goal"])
    assert PL.fingerprint(a) != PL.fingerprint(b) and len(PL.fingerprint(a)) == 64


# ---- the proof workloads of bench.py (scenes.PROOF_CONFIGS) ---------------------------------------------------
def _solve_proof_workload(name):
    from paper_2406_04795_b200 import pipeline as PL, scenes
    conf = scenes.PROOF_CONFIGS[name]
    pdict = scenes.fence_problem_dict(conf["dof"], clutter=conf["clutter"], **conf.get("scene", {}))
    problem = PL.problem_file_from_dict(pdict).problem()
    out = PL.solve(problem, PL.SolveParams(timeout=600.0, **conf["params"]))
    return problem, out


@pytest.mark.gpu
def test_fence_twin_matches_the_reference_solve():
    """`dof3-proof`, the 3-DoF twin of the fence scenes: the reference's own solve() on the same problem file and parameters
    (profiles/r2_reference_dof3_proof.json, 52 s on the CPU) ends after 3 iterations with 1984 coarse edges, 3002 cells,
    7877 certificate points and 2305 support vectors -- so must this one, and the certificate must verify."""
    from paper_2406_04795_b200 import pipeline as PL
    problem, out = _solve_proof_workload("dof3-proof")
    assert isinstance(out, PL.InfeasibilityProof)
    assert int(out.meta["iterations"]) == 3
    assert (out.coarse_edges, out.coarse_cells, out.points.shape[0], out.manifold.support.shape[0]) == (1984, 3002, 7877, 2305)
    assert [r.get("roadmap") for r in out.stats.iterations] == [602, 1643, 2305]
    assert PL.verify_proof(out, problem).ok


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["dof4-proof", "dof5-proof"])
def test_high_dof_infeasibility_proofs(name):
    """BASELINE configs 2-3: the whole outer loop on a 4- / 5-DoF arm behind a fence, with clutter: it must end in an
    InfeasibilityProof with no free point among its collision-checked points, accepted by verify_proof incl. the
    reconstruction check (re-trace + re-refinement from the certificate alone)."""
    from paper_2406_04795_b200 import pipeline as PL
    problem, out = _solve_proof_workload(name)
    assert isinstance(out, PL.InfeasibilityProof), getattr(out, "reason", out)
    assert out.closure_ok and out.points.shape[0] > 100_000 and out.points.shape[1] == problem.dof
    last = out.stats.iterations[-1]
    assert last["free_points"] == 0 and last["points"] == out.points.shape[0]
    report = PL.verify_proof(out, problem)
    assert report.ok, report.first_failure()
    assert [c.name for c in report.checks][-1] == "reconstruction"
