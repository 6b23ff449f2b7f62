"""verify_proof on the device path (first "next" row) against the REAL reference:
tests/golden/proof.npz holds a certificate produced by the reference's own solve() on its bundled wall2d
scene, and the reference's verify_proof() verdicts for the intact certificate and a tamper matrix
(tests/golden/make_golden.py::proof_golden).  The product must return the same checks, in the same order,
with the same verdicts."""

from __future__ import annotations

import copy
import json

import numpy as np
import pytest

from tests.conftest import Golden


def _problem_and_proof(g):
    import paper_2406_04795_b200 as P
    from paper_2406_04795_b200 import collision as CO, manifold as M, pipeline as PL
    rs = json.loads(str(g["robot_scene_json"][0]))
    robot, scene = CO.robot_from_dict(rs["robot"]), CO.scene_from_dict(rs["scene"])
    problem = PL.Problem(robot, scene, g["start"], g["goal"])
    n = g["support"].shape[1]
    bar = g["barrier"]
    barrier = M.BoxBarrier(bar[2:2 + n], bar[2 + n:], bar[0], bar[1])
    manifold = M.KernelClassifierManifold(g["support"], g["weights"], g["gbb"][0], g["gbb"][1], barrier=barrier)
    lam, k, eps, f_start, f_goal, ce, cc, closure, poly = g["params"]
    proof = PL.InfeasibilityProof(manifold=manifold, lam=float(lam), k=int(k), eps=float(eps), points=g["points"].copy(),
                                  f_start=float(f_start), f_goal=float(f_goal), fingerprint=str(g["fingerprint"][0]),
                                  closure_ok=bool(closure), polyline_closed=None if poly < 0 else bool(poly),
                                  coarse_edges=int(ce), coarse_cells=int(cc))
    return problem, proof


def _tampered(proof, problem, kind):
    from paper_2406_04795_b200 import manifold as M
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
        m = proof.manifold
        p.manifold = M.KernelClassifierManifold(m.support, m.weights, m.gamma, m.bias + 0.05, barrier=m.barrier)
    elif kind == "point_free":
        p.points = proof.points.copy(); p.points[0] = problem.q_start
    return p


def test_fingerprint_matches_the_reference_serialization():
    """CPU: the canonical robot+scene JSON and its SHA-256 equal the reference's (pipeline.py:110-117)."""
    from paper_2406_04795_b200 import collision as CO, pipeline as PL
    g = Golden("proof")
    rs = json.loads(str(g["robot_scene_json"][0]))
    robot, scene = CO.robot_from_dict(rs["robot"]), CO.scene_from_dict(rs["scene"])
    assert {"robot": CO.robot_to_dict(robot), "scene": CO.scene_to_dict(scene)} == rs

    class _P:
        pass
    p = _P(); p.robot, p.scene = robot, scene
    assert PL.fingerprint(p) == str(g["fingerprint"][0])


@pytest.mark.gpu
def test_verify_proof_verdicts_equal_the_reference():
    from paper_2406_04795_b200 import pipeline as PL
    g = Golden("proof")
    problem, proof = _problem_and_proof(g)
    for kind, names, passed in zip(g["tamper_kinds"], g["tamper_check_names"], g["tamper_check_passed"]):
        rep = PL.verify_proof(_tampered(proof, problem, str(kind)), problem)
        assert [c.name for c in rep.checks] == json.loads(str(names)), kind
        assert [bool(c.passed) for c in rep.checks] == json.loads(str(passed)), (kind, rep.first_failure())
    rep = PL.verify_proof(proof, problem)
    assert rep.ok and rep.checks[-1].name == "reconstruction" and "155 points reproduced" in rep.checks[-1].detail
    assert PL.verify_proof(proof, problem, reconstruct=False).ok


@pytest.mark.gpu
def test_reconstruction_reproduces_the_stored_points():
    """The re-trace seeded at the certificate's own points + re-refinement (device path) returns the reference's
    point set to the north-star tolerance."""
    import paper_2406_04795_b200 as P
    from paper_2406_04795_b200 import subdivision as S, tracer as T, lattice as L
    g = Golden("proof")
    problem, proof = _problem_and_proof(g)
    cfg = T.TraceConfig(lattice=L.LatticeConfig(2, proof.lam * proof.k), max_edges=4 * proof.coarse_edges + 1024, eps=proof.eps)
    res = T.trace(proof.points, proof.manifold, cfg)
    assert res.closure_ok and len(res.edges) == proof.coarse_edges
    cells = S.coarse_cells(res)
    assert len(cells) == proof.coarse_cells
    ref = S.refine(cells, S.build_template(2, proof.k), proof.manifold, lambda pts: np.ones(len(pts), dtype=bool), cfg)
    assert ref.points.shape == proof.points.shape
    assert np.allclose(ref.points, proof.points, rtol=1e-5, atol=1e-8)
