"""The slice of ``permatrace/pipeline.py`` that sits on the hot path, and its two callers.

`Problem` (pipeline.py:80-107), the non-free checker the refinement stage calls (pipeline.py:256-270), and the
"next" rows of SURVEY.md section 8f: the certificate verifier `verify_proof` (pipeline.py:464-580), whose expensive
part re-runs trace + coarse_cells + refine on the device path, and the learn -> trace -> refine -> check loop `solve`
(pipeline.py:284-430) with the roadmap of `planner.py` feeding it.  The text formats (INFPROOF / KCLF / EDGEMESH) stay in
the reference package; INTEGRATION.md shows how they bind to this module.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
import warnings
from dataclasses import dataclass, field

import numpy as np

from .collision import (RobotModel, Scene, _check, config_in_collision, device_checker, joint_limits, robot_to_dict,
                        scene_to_dict)

__all__ = ["Problem", "not_free_checker", "_not_free_checker", "fingerprint", "InfeasibilityProof", "CheckResult",
           "VerifyReport", "verify_proof", "ProblemFile", "load_problem_file", "SolveParams", "SolveStats", "Plan",
           "SolveTimeout", "solve"]


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


# ---- scene files and solve parameters (reference pipeline.py:120-208) -----------------------------------

_SCENE_PARAM_KEYS = {
    "lambda": ("lam", float), "k": ("k", int), "eps": ("eps", float), "gamma": ("gamma", float),
    "seeds": ("seeds", int), "samples": ("samples_per_iter", int), "margin": ("trace_margin", float),
    "regularization": ("regularization", float), "push": ("push", float),
}


@dataclass
class SolveParams:
    """Resolution and budget knobs of `solve`; same fields and defaults as the reference (pipeline.py:172-205).
    `push=None` means lam * sqrt(2 gamma) (about one fine cell into the blocked side), `trace_margin=None` the
    reference's box inflation rule."""

    lam: float = 0.05
    k: int = 2
    eps: float = 1e-9
    seeds: int = 20
    seed_tol: float = 1e-8
    memory_budget: int = 64 * 2**20
    rng_seed: int = 0
    workers: int = 1
    samples_per_iter: int = 500
    max_iters: int = 50
    timeout: float = 300.0
    gamma: float | None = None
    regularization: float = 1e-3
    push: float | None = None
    knn: int = 10
    max_edges: int = 10_000_000
    trace_margin: float | None = None
    # not in the reference: at most this many free points of one iteration go back into the roadmap (an even spread over
    # the refinement order).  None = all of them, the reference's behaviour.  At 5-6 DoF one early iteration can return
    # 10^5-10^6 free points, and every roadmap vertex is a support vector of the next classifier.
    feedback_cap: int | None = None

    def __post_init__(self):
        if self.lam <= 0 or self.k < 1 or self.eps <= 0:
            raise ValueError("lam, k and eps must be positive")
        if self.seeds < 1 or self.samples_per_iter < 1 or self.max_iters < 1:
            raise ValueError("seeds, samples_per_iter and max_iters must be positive")


@dataclass
class ProblemFile:
    """Parsed scene file: models plus optional suggested endpoints / parameters (pipeline.py:120-156)."""

    robot: RobotModel
    scene: Scene
    start: np.ndarray | None
    goal: np.ndarray | None
    params: dict

    def problem(self, start=None, goal=None) -> Problem:
        start = self.start if start is None else start
        goal = self.goal if goal is None else goal
        if start is None or goal is None:
            raise ValueError("scene file has no endpoints; pass --start/--goal")
        return Problem(self.robot, self.scene, start, goal)

    def solve_params(self, **overrides) -> SolveParams:
        """SolveParams from the file's params block; keyword overrides win."""
        params = SolveParams()
        for key, value in self.params.items():
            if key not in _SCENE_PARAM_KEYS:
                raise ValueError(f"unknown scene parameter {key!r}")
            attr, cast = _SCENE_PARAM_KEYS[key]
            setattr(params, attr, cast(value))
        for attr, value in overrides.items():
            if not hasattr(params, attr):
                raise ValueError(f"unknown solve parameter {attr!r}")
            setattr(params, attr, value)
        params.__post_init__()
        return params


def problem_file_from_dict(data, origin: str = "<dict>") -> ProblemFile:
    from .collision import robot_from_dict, scene_from_dict
    if not isinstance(data, dict) or "robot" not in data or "scene" not in data:
        raise ValueError(f"{origin}: expected top-level robot: and scene: sections")
    prob = data.get("problem") or {}
    start = np.asarray(prob["start"], dtype=np.float64) if "start" in prob else None
    goal = np.asarray(prob["goal"], dtype=np.float64) if "goal" in prob else None
    return ProblemFile(robot_from_dict(data["robot"]), scene_from_dict(data["scene"]), start, goal,
                       dict(prob.get("params") or {}))


def load_problem_file(path) -> ProblemFile:
    """YAML scene file in the reference schema (pipeline.py:159-168)."""
    import yaml
    with open(path) as fh:
        return problem_file_from_dict(yaml.safe_load(fh), str(path))


@dataclass
class SolveStats:
    iterations: list = field(default_factory=list)
    outcome: str = ""
    seconds: float = 0.0


@dataclass
class Plan:
    """Collision-free path, validated at half the roadmap step."""

    path: list
    stats: SolveStats


@dataclass
class SolveTimeout:
    reason: str
    stats: SolveStats


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


def _set_gap(a: np.ndarray, b: np.ndarray, tol: float = 0.0) -> float:
    """Symmetric Hausdorff distance of two point sets.  Both come out of the same deterministic pipeline, so the
    row-wise comparison normally settles it; otherwise nearest neighbours by KD-tree like the reference."""
    if a.shape == b.shape:
        rowwise = float(np.max(np.linalg.norm(a - b, axis=1)))      # an upper bound of the Hausdorff distance
        if rowwise <= tol:
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
    from ._cabi import RangeError
    try:
        result = trace(points, manifold, cfg)
    except RangeError as exc:        # the zero set leaves the packed-key window of the device tracer: a failed check, not a crash
        return CheckResult(name, False, f"re-trace not representable on the device: {exc}")
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
    gap = _set_gap(refined.points, points, tol)
    if gap > tol:
        return CheckResult(name, False, f"point sets differ by {gap:.3g} > {tol:.3g}")
    return CheckResult(name, True, f"{points.shape[0]} points reproduced within {tol:.3g}")


# ---- the solve loop (reference pipeline.py:272-430) ----------------------------------------------------

def _drop_blocked_segment(roadmap, path) -> bool:
    """Re-validate a found path at half step; cut the first failing roadmap edge (pipeline.py:272-281)."""
    i = roadmap.first_blocked_segment(path, roadmap.delta / 2.0)
    if i is None:
        return False
    u, v = roadmap.index_of(path[i]), roadmap.index_of(path[i + 1])
    roadmap.neighbors[u].pop(v, None)
    roadmap.neighbors[v].pop(u, None)
    return True


def _learn_manifold(labels, lo, hi, params: SolveParams):
    """Separating field of one iteration: ridge classifier + limit-box barrier + bias push (pipeline.py:327-349).
    Returns (manifold, gamma, sigma)."""
    from .manifold import BoxBarrier, KernelClassifierManifold, median_gamma, train_classifier
    gamma = params.gamma
    if gamma is None:
        gamma = median_gamma(np.vstack([labels.positive, labels.negative]))
    sigma = 1.0 / np.sqrt(2.0 * gamma)
    barrier = BoxBarrier(lo, hi, scale=sigma / 4.0, gain=2.0 / sigma)
    manifold = train_classifier(labels.positive, labels.negative, gamma=gamma, regularization=params.regularization,
                                barrier=barrier)
    push = params.lam * np.sqrt(2.0 * gamma) if params.push is None else params.push
    if push:
        manifold = KernelClassifierManifold(manifold.support, manifold.weights, manifold.gamma,
                                            bias=manifold.bias + push, barrier=barrier,
                                            train_accuracy=manifold.train_accuracy)
    return manifold, gamma, sigma


def solve(problem: Problem, params: SolveParams | None = None):
    """Search for a `Plan` or an `InfeasibilityProof`; `SolveTimeout` when neither (reference pipeline.py:284-430).

    Same loop, same random stream (one generator shared by the roadmap and the seed sampler, consumed in the
    reference's order), same per-iteration record keys.  The roadmap's collision work goes to the device in one
    batch per `grow` / `insert_free_points`, seeds are projected in one batched Newton iteration, and trace,
    coarse_cells, refine, the non-free labels and the self-verification run on the device path.
    """
    from .lattice import LatticeConfig
    from .manifold import sample_seeds
    from .planner import Roadmap, find_path, grow, insert_free_points, labeled_samples
    from .subdivision import build_template, coarse_cells, refine
    from .tracer import TraceConfig, trace
    from ._cabi import RangeError

    params = params or SolveParams()
    t0 = time.perf_counter()
    deadline = t0 + params.timeout
    stats = SolveStats()
    n = problem.dof
    lo, hi = problem.limits()
    rng = np.random.default_rng(params.rng_seed)
    roadmap = Roadmap(problem.robot, problem.scene, delta=params.lam / 4.0, knn=params.knn, rng=rng)
    roadmap.add_config(problem.q_start, free=True)
    roadmap.add_config(problem.q_goal, free=True)
    template = build_template(n, params.k)
    coarse = params.lam * params.k
    scene_id = fingerprint(problem)

    def finish(outcome: str, value):
        stats.outcome = outcome
        stats.seconds = time.perf_counter() - t0
        return value

    live_log = os.environ.get("PERMATRACE_B200_SOLVE_LOG", "") not in ("", "0")
    for iteration in range(1, params.max_iters + 1):
        if live_log and stats.iterations:      # the finished record of the previous iteration, as it happens
            print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in stats.iterations[-1].items()}),
                  file=sys.stderr, flush=True)
        record: dict = {"iteration": iteration}
        stats.iterations.append(record)
        if time.perf_counter() > deadline:
            return finish("timeout", SolveTimeout("wall-clock timeout", stats))
        grow(roadmap, params.samples_per_iter)
        record["roadmap"] = len(roadmap)
        path = find_path(roadmap, problem.q_start, problem.q_goal)
        while path is not None and _drop_blocked_segment(roadmap, path):
            path = find_path(roadmap, problem.q_start, problem.q_goal)
        if path is not None:
            return finish("plan", Plan([np.asarray(q) for q in path], stats))
        labels = labeled_samples(roadmap, problem.q_start)
        record["positive"], record["negative"] = len(labels.positive), len(labels.negative)
        if len(labels.positive) == 0 or len(labels.negative) == 0:
            continue

        t = time.perf_counter()
        manifold, gamma, sigma = _learn_manifold(labels, lo, hi, params)
        record["train_s"] = time.perf_counter() - t
        margin = params.trace_margin
        if margin is None:
            margin = max(3.0 * coarse, 2.0 * sigma + (1.0 + 2.0 * np.sqrt(n)) * coarse)
        cfg = TraceConfig(lattice=LatticeConfig(n, coarse), box=(tuple(lo - margin), tuple(hi + margin)),
                          max_edges=params.max_edges, workers=params.workers, eps=params.eps)
        f_start, f_goal = (float(v) for v in manifold.values(np.stack([problem.q_start, problem.q_goal])))
        if (f_start > 0.0) == (f_goal > 0.0):
            record["skip"] = "no separation"
            continue
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")            # sparse zero sets fail many draws
            seeds = sample_seeds(manifold, (lo, hi), params.seeds, tol=params.seed_tol, rng=rng,
                                 min_separation=coarse / 2.0)
        if seeds.shape[0] == 0:
            record["skip"] = "no seeds"
            continue

        t = time.perf_counter()
        try:
            result = trace(seeds, manifold, cfg)
        except RangeError as exc:    # lattice too fine for the packed keys at this dimension: skip the iteration, say why
            record["skip"] = f"trace out of key range: {exc}"
            continue
        record["trace_s"] = time.perf_counter() - t
        record["edges"] = len(result.edges)
        if not len(result.edges) or not result.closure_ok:
            record["skip"] = "trace not closed"
            record["dropped"] = result.stats.dropped_out_of_box
            record["complete"] = result.stats.complete
            continue
        cells = coarse_cells(result)
        record["cells"] = len(cells)
        check_times: list = []
        checker = _not_free_checker(problem, check_times)
        t = time.perf_counter()
        refined = refine(cells, template, manifold, checker, cfg, memory_budget=params.memory_budget)
        record["refine_s"] = time.perf_counter() - t
        record["check_s"] = float(sum(check_times))
        record["points"] = int(refined.points.shape[0])
        record["crossing_edges"] = int(sum(b.crossing_edges for b in refined.batch_stats))   # (not a reference key)
        record["free_points"] = int(refined.free_points.shape[0])
        if refined.free_points.shape[0]:
            # the zero set still touches free space: feed those configurations back into the roadmap
            feedback = refined.free_points
            if os.environ.get("PERMATRACE_B200_SOLVE_LOG", "") == "2":       # diagnostics only: where the free points are
                record["free_lo"] = [round(float(v), 3) for v in feedback.min(axis=0)]
                record["free_hi"] = [round(float(v), 3) for v in feedback.max(axis=0)]
            if params.feedback_cap is not None and feedback.shape[0] > params.feedback_cap:
                feedback = feedback[np.linspace(0, feedback.shape[0] - 1, params.feedback_cap).astype(np.int64)]
            record["fed_back"] = insert_free_points(roadmap, feedback, dedup_tol=params.lam / 4.0)
            continue
        if refined.points.shape[0] == 0:
            record["skip"] = "empty refinement"
            continue

        proof = InfeasibilityProof(
            manifold=manifold, lam=params.lam, k=params.k, eps=params.eps, points=np.array(refined.points),
            f_start=f_start, f_goal=f_goal, fingerprint=scene_id, closure_ok=result.stats.closure_ok,
            polyline_closed=result.stats.polyline_closed, coarse_edges=len(result.edges), coarse_cells=len(cells),
            meta={"generator": "permatrace-b200", "iterations": str(iteration), "support": str(manifold.support.shape[0])})
        report = verify_proof(proof, problem)
        if report.ok:
            proof.stats = stats
            return finish("proof", proof)
        record["skip"] = "self-verification failed: " + report.first_failure()
    return finish("timeout", SolveTimeout("iteration budget exhausted", stats))
