"""The slice of ``permatrace/pipeline.py`` that sits on the hot path.

`Problem` (pipeline.py:80-107), the non-free checker the refinement stage calls (pipeline.py:256-270)
and -- the first "next" row of SURVEY.md section 8f -- the certificate verifier `verify_proof`
(pipeline.py:464-580), whose expensive part re-runs trace + coarse_cells + refine on the device path.
The solve loop and the text formats stay in the reference package; INTEGRATION.md shows how they bind
to this module.
"""

from __future__ import annotations

import hashlib
import json
import time
from dataclasses import dataclass, field

import numpy as np

from .collision import (RobotModel, Scene, _check, config_in_collision, device_checker, joint_limits, robot_to_dict,
                        scene_to_dict)

__all__ = ["Problem", "not_free_checker", "_not_free_checker", "fingerprint", "InfeasibilityProof", "CheckResult",
           "VerifyReport", "verify_proof"]


@dataclass
class Problem:
    """Scene + robot + endpoints; endpoints must be inside the limits and collision-free."""

    robot: RobotModel
    scene: Scene
    q_start: np.ndarray
    q_goal: np.ndarray

    def __post_init__(self):
        self.q_start = np.asarray(self.q_start, dtype=np.float64)
        self.q_goal = np.asarray(self.q_goal, dtype=np.float64)
        n = self.robot.dof
        if self.q_start.shape != (n,) or self.q_goal.shape != (n,):
            raise ValueError(f"start/goal must have {n} coordinates")
        lo, hi = joint_limits(self.robot)
        for name, q in (("start", self.q_start), ("goal", self.q_goal)):
            if np.any(q < lo) or np.any(q > hi):
                raise ValueError(f"{name} configuration violates the joint limits")
            if config_in_collision(q, self.robot, self.scene):
                raise ValueError(f"{name} configuration is in collision")

    @property
    def dof(self) -> int:
        return self.robot.dof

    def limits(self):
        return joint_limits(self.robot)


class _DeviceNotFreeChecker:
    """(m, n) float64 -> bool[m]: outside the joint-limit box, or in collision.

    Callable like the reference's closure; `device_checker` lets `refine` label the points with
    ``pt_check_kernel`` (mode PT_LIMIT_UNFREE) without copying them to the host first.
    """

    def __init__(self, robot: RobotModel, scene: Scene, accumulator: list | None = None):
        self.robot = robot
        self.scene = scene
        self.accumulator = accumulator
        self.device_checker = device_checker(robot, scene)

    def __call__(self, points) -> np.ndarray:
        t0 = time.perf_counter()
        pts = np.atleast_2d(np.asarray(points, dtype=np.float64))
        out = _check(pts, self.robot, self.scene, 1)
        if self.accumulator is not None:
            self.accumulator.append(time.perf_counter() - t0)
        return out


def _not_free_checker(problem, accumulator: list | None = None):
    """Reference name and signature (pipeline.py:256); `problem` needs .robot and .scene."""
    return _DeviceNotFreeChecker(problem.robot, problem.scene, accumulator)


not_free_checker = _not_free_checker


# ---- certificates (reference pipeline.py:110-117, :232-253, :434-580) -----------------------------

def fingerprint(problem) -> str:
    """SHA-256 over the canonical robot+scene serialization (pipeline.py:110-117)."""
    canon = json.dumps({"robot": robot_to_dict(problem.robot), "scene": scene_to_dict(problem.scene)},
                       sort_keys=True, separators=(",", ":"))
    return hashlib.sha256(canon.encode()).hexdigest()


@dataclass
class InfeasibilityProof:
    """Same fields as the reference certificate (pipeline.py:232-253); any object with these attributes
    (e.g. the reference's own dataclass) is accepted by `verify_proof`."""

    manifold: object
    lam: float
    k: int
    eps: float
    points: np.ndarray
    f_start: float
    f_goal: float
    fingerprint: str
    closure_ok: bool
    polyline_closed: bool | None
    coarse_edges: int
    coarse_cells: int
    meta: dict = field(default_factory=dict)


@dataclass
class CheckResult:
    name: str
    passed: bool
    detail: str


@dataclass
class VerifyReport:
    checks: list

    @property
    def ok(self) -> bool:
        return all(c.passed for c in self.checks)

    def first_failure(self) -> str:
        for c in self.checks:
            if not c.passed:
                return f"{c.name}: {c.detail}"
        return ""


def _device_manifold(m):
    """The certificate's manifold as a device-capable KernelClassifierManifold (the reference's own class is
    accepted: support / weights / gamma / bias / barrier are read off it)."""
    from .manifold import BoxBarrier, ImplicitManifold, KernelClassifierManifold
    if isinstance(m, ImplicitManifold):
        return m
    barrier = getattr(m, "barrier", None)
    if barrier is not None and not isinstance(barrier, BoxBarrier):
        barrier = BoxBarrier(barrier.lower, barrier.upper, barrier.scale, barrier.gain)
    return KernelClassifierManifold(m.support, m.weights, m.gamma, m.bias, barrier=barrier)


def _gradient_norms(manifold, points: np.ndarray) -> np.ndarray:
    """|grad F| at every point (pipeline.py:457-461); learned manifolds in one device batch, analytic test
    manifolds through their closed forms."""
    if hasattr(manifold, "gradients"):
        return np.linalg.norm(manifold.gradients(points), axis=1)
    out = np.empty(points.shape[0])
    for i, q in enumerate(points):
        out[i] = float(np.linalg.norm(manifold.gradient(q)))
    return out


def verify_proof(proof, problem, reconstruct: bool = True) -> VerifyReport:
    """Independent certificate check, same checks / order / early exits as the reference
    (pipeline.py:464-536); field values, collision labels and the whole re-trace + re-refinement run on
    the device path."""
    checks: list = []
    m = _device_manifold(proof.manifold)
    points = np.asarray(proof.points, dtype=np.float64)

    expected = fingerprint(problem)
    checks.append(CheckResult("fingerprint", proof.fingerprint == expected,
                              f"stored {proof.fingerprint[:12]}.., scene has {expected[:12]}.."))
    if m.dim != problem.dof or points.ndim != 2 or points.shape[1] != problem.dof:
        checks.append(CheckResult("dimensions", False,
                                  f"manifold dim {m.dim}, points {points.shape}, robot dof {problem.dof}"))
        return VerifyReport(checks)

    f_start, f_goal = (float(v) for v in m.values(np.stack([problem.q_start, problem.q_goal])))
    separated = (f_start > 0.0) != (f_goal > 0.0)
    stored_ok = (abs(f_start - proof.f_start) <= 1e-9 * max(1.0, abs(f_start))
                 and abs(f_goal - proof.f_goal) <= 1e-9 * max(1.0, abs(f_goal)))
    checks.append(CheckResult("separation", separated and stored_ok,
                              f"F(start)={f_start:.6g}, F(goal)={f_goal:.6g}, stored ({proof.f_start:.6g}, {proof.f_goal:.6g})"))
    if points.shape[0] == 0:
        checks.append(CheckResult("points", False, "certificate has no points"))
        return VerifyReport(checks)

    not_free = _not_free_checker(problem)(points)
    checks.append(CheckResult("points non-free", bool(not_free.all()),
                              f"{int((~not_free).sum())} of {len(points)} points are free"))

    residuals = np.abs(m.values(points))
    tolerance = 4.0 * proof.eps * (_gradient_norms(m, points) + 1e-12)
    on_manifold = residuals <= tolerance
    worst = int(np.argmax(residuals - tolerance))
    checks.append(CheckResult("points on zero set", bool(on_manifold.all()),
                              f"worst |F|={residuals[worst]:.3g} vs tol {tolerance[worst]:.3g}"))

    flags_ok = bool(proof.closure_ok) and (proof.polyline_closed is not False)
    checks.append(CheckResult("closure flags", flags_ok,
                              f"closure_ok={proof.closure_ok}, polyline_closed={proof.polyline_closed}"))

    if reconstruct and all(c.passed for c in checks):
        checks.append(_reconstruction_check(proof, m, points))
    return VerifyReport(checks)


def _set_gap(a: np.ndarray, b: np.ndarray) -> float:
    """Symmetric Hausdorff distance of two point sets.  Both come out of the same deterministic pipeline, so the
    row-wise comparison normally settles it; otherwise nearest neighbours by KD-tree like the reference."""
    if a.shape == b.shape:
        rowwise = float(np.max(np.linalg.norm(a - b, axis=1)))
        if rowwise <= 1e-6:
            return rowwise
    from scipy.spatial import cKDTree
    return float(max(cKDTree(a).query(b)[0].max(), cKDTree(b).query(a)[0].max()))


def _reconstruction_check(proof, manifold, points: np.ndarray) -> CheckResult:
    """Re-derive the certificate from its own manifold and parameters, seeding the trace at the stored points
    (pipeline.py:539-580): same counts, same point set within 64 eps."""
    from .lattice import LatticeConfig
    from .subdivision import build_template, coarse_cells, refine
    from .tracer import TraceConfig, trace
    name = "reconstruction"
    n = points.shape[1]
    cfg = TraceConfig(lattice=LatticeConfig(n, proof.lam * proof.k), max_edges=4 * proof.coarse_edges + 1024,
                      workers=1, eps=proof.eps)
    result = trace(points, manifold, cfg)
    if not result.closure_ok:
        return CheckResult(name, False, "re-trace did not close")
    if len(result.edges) != proof.coarse_edges:
        return CheckResult(name, False, f"re-trace found {len(result.edges)} coarse edges, recorded {proof.coarse_edges}")
    cells = coarse_cells(result)
    if len(cells) != proof.coarse_cells:
        return CheckResult(name, False, f"re-trace found {len(cells)} coarse cells, recorded {proof.coarse_cells}")
    template = build_template(n, proof.k)
    refined = refine(cells, template, manifold, lambda pts: np.ones(len(pts), dtype=bool), cfg)
    if refined.points.shape[0] != points.shape[0]:
        return CheckResult(name, False, f"re-refinement produced {refined.points.shape[0]} points, stored {points.shape[0]}")
    tol = max(64.0 * proof.eps, 1e-12)
    gap = _set_gap(refined.points, points)
    if gap > tol:
        return CheckResult(name, False, f"point sets differ by {gap:.3g} > {tol:.3g}")
    return CheckResult(name, True, f"{points.shape[0]} points reproduced within {tol:.3g}")
