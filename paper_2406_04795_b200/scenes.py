"""Synthetic 3/4/5/6-DoF manipulator scenes in the reference's dict/YAML schema.

The reference ships only 2-DoF point robots and the 3-DoF ``arm3wall`` (permatrace/scenes/*.yaml);
BASELINE.json's configs 2-5 need 4/5/6-DoF arms.  These follow the arm3wall pattern extended
(SURVEY.md section 8d): a serial chain of revolute joints alternating z / y axes, link length 0.4,
four collision spheres of radius 0.06 per link, box / cylinder / sphere obstacles.  The dicts load
through ``collision.robot_from_dict`` / ``scene_from_dict`` here and in the reference alike.
"""

from __future__ import annotations

import numpy as np

__all__ = ["arm_robot_dict", "arm_scene_dict", "synthetic_support", "BENCH_CONFIGS", "fence_problem_dict", "PROOF_CONFIGS"]


def arm_robot_dict(dof: int, limit: float = 1.5, link: float = 0.4, spheres_per_link: int = 4,
                   radius: float = 0.06) -> dict:
    joints = []
    for j in range(dof):
        joints.append({
            "type": "revolute",
            "axis": [0, 0, 1] if j % 2 == 0 else [0, 1, 0],
            "origin": {"xyz": [0.0 if j == 0 else link, 0.0, 0.0], "rpy": [0, 0, 0]},
            "limits": [-limit, limit],
        })
    spheres = []
    for j in range(1, dof + 1):
        for s in range(1, spheres_per_link + 1):
            spheres.append({"link": j, "offset": [link * s / spheres_per_link, 0.0, 0.0], "radius": radius})
    return {"joints": joints, "spheres": spheres}


def arm_scene_dict(n_obstacles: int = 8, seed: int = 7, reach: float = 2.0) -> dict:
    """Deterministic clutter of boxes, cylinders and spheres in a shell around the arm's base."""
    rng = np.random.default_rng(seed)
    obstacles = []
    for i in range(n_obstacles):
        direction = rng.normal(size=3)
        direction /= np.linalg.norm(direction)
        centre = direction * rng.uniform(0.45 * reach, 0.9 * reach)
        rpy = rng.uniform(-0.6, 0.6, size=3)
        origin = {"xyz": [float(v) for v in centre], "rpy": [float(v) for v in rpy]}
        kind = i % 4
        if kind in (0, 1):
            size = rng.uniform(0.25, 0.7, size=3)
            obstacles.append({"type": "box", "size": [float(v) for v in size], "origin": origin})
        elif kind == 2:
            obstacles.append({"type": "cylinder", "height": float(rng.uniform(0.4, 1.0)),
                              "radius": float(rng.uniform(0.1, 0.3)), "origin": origin})
        else:
            obstacles.append({"type": "sphere", "radius": float(rng.uniform(0.15, 0.35)), "origin": origin})
    return {"obstacles": obstacles}


def synthetic_support(n: int, count: int, r_split: float, limit: float = 1.5, seed: int = 0):
    """Appendix-B recipe of SURVEY.md: support ~ U(limits), positive class = ||x|| < r_split."""
    rng = np.random.default_rng(seed)
    x = rng.uniform(-limit, limit, size=(count, n))
    inside = np.linalg.norm(x, axis=1) < r_split
    return x[inside], x[~inside], rng


# name -> parameters of the benchmark / parity workloads (BASELINE.json configs 1-5 shapes)
BENCH_CONFIGS = {
    "dof3": dict(n=3, support=512, lam=0.2, r_split=0.9, obstacles=3),
    "dof4": dict(n=4, support=1024, lam=0.3, r_split=0.9, obstacles=3),
    "dof5": dict(n=5, support=1024, lam=0.4, r_split=0.9, obstacles=8),
    "dof6": dict(n=6, support=2048, lam=0.35, r_split=1.3, obstacles=8),
    "dof6-stress": dict(n=6, support=2048, lam=0.2, r_split=1.3, obstacles=48),
    # BASELINE.json config 5 at its stated size: ~10^9 simplices (crossings grow like lambda^-5)
    "dof6-stress1g": dict(n=6, support=2048, lam=0.175, r_split=1.3, obstacles=48),
    # support set of the size the reference's own solve loop ends with (arm3wall: 4 199 roadmap samples)
    "dof6-s4096": dict(n=6, support=4096, lam=0.35, r_split=1.3, obstacles=8),
    # the support-set size the SURVEY expects for real 6-DoF proofs (10^3..10^4 roadmap samples): 8 support chunks
    "dof6-s16384": dict(n=6, support=16384, lam=0.35, r_split=1.3, obstacles=8),
}


# ---- infeasible 4/5/6-DoF problems (BASELINE.json configs 3-4: "full infeasibility proof") ------------------------------
def fence_problem_dict(dof: int, clutter: int = 6, seed: int = 11, q1_limit: float = 2.4, limit: float = 1.2,
                       link: float = 0.4, radius: float = 0.06) -> dict:
    """The reference's arm3wall pattern (permatrace/scenes/arm3wall.yaml) extended to `dof` joints: the base link must
    sweep past a radial fence on the +x axis to get from pointing +y to pointing -y, and joint 1 stops short of a full
    turn, so there is no way around.  The fence only ever touches link 1 (it is low and close to the base), so the
    blocked region is a slab in q1 for every posture of the other joints; `clutter` further boxes / cylinders / spheres sit
    where the distal links reach them, which dents the free space without reconnecting it.  Returns a problem-file dict in
    the reference's schema (`pipeline.problem_file_from_dict`, reference pipeline.py:120-168)."""
    joints = []
    for j in range(dof):
        joints.append({
            "type": "revolute",
            "axis": [0, 0, 1] if j % 2 == 0 else [0, 1, 0],
            "origin": {"xyz": [0.0 if j == 0 else link, 0.0, 0.0], "rpy": [0, 0, 0]},
            "limits": [-q1_limit, q1_limit] if j == 0 else [-limit, limit],
        })
    spheres = [{"link": j, "offset": [link * s / 4, 0.0, 0.0], "radius": radius}
               for j in range(1, dof + 1) for s in range(1, 5)]
    obstacles = [{"type": "box", "size": [0.18, 0.30, 0.20], "origin": {"xyz": [0.31, 0.0, 0.0], "rpy": [0, 0, 0]}}]
    rng = np.random.default_rng(seed)
    reach = link * dof
    for i in range(clutter):
        # a shell the distal links sweep through, kept away from the base so that link 1 never meets it
        ang, height = rng.uniform(-np.pi, np.pi), rng.uniform(-0.5, 0.5) * reach
        rad = rng.uniform(0.62, 0.95) * reach
        origin = {"xyz": [float(rad * np.cos(ang)), float(rad * np.sin(ang)), float(height)],
                  "rpy": [float(v) for v in rng.uniform(-0.5, 0.5, size=3)]}
        kind = i % 3
        if kind == 0:
            obstacles.append({"type": "box", "size": [float(v) for v in rng.uniform(0.15, 0.35, size=3)], "origin": origin})
        elif kind == 1:
            obstacles.append({"type": "cylinder", "height": float(rng.uniform(0.3, 0.6)), "radius": float(rng.uniform(0.08, 0.16)),
                              "origin": origin})
        else:
            obstacles.append({"type": "sphere", "radius": float(rng.uniform(0.1, 0.2)), "origin": origin})
    start = [0.5 * np.pi] + [0.0] * (dof - 1)
    goal = [-0.5 * np.pi] + [0.0] * (dof - 1)
    return {"robot": {"joints": joints, "spheres": spheres}, "scene": {"obstacles": obstacles},
            "problem": {"start": start, "goal": goal}}


# name -> (problem generator arguments, SolveParams overrides) of the end-to-end proof workloads.  Parameters found on the
# B200 (gpurun_out logs summarised in profiles/r2_proof_*.json): a wide kernel (small gamma) keeps the learned surface
# smooth, the push stays below 1 (labels are +-1, a larger bias offset erases the sign change between start and goal:
# "no separation"), and the feedback cap keeps the support set -- every roadmap vertex -- in the 10^4 range.
def _push(lam, gamma, mult):
    return mult * lam * float(np.sqrt(2.0 * gamma))


PROOF_CONFIGS = {
    "dof4-proof": dict(dof=4, clutter=3, params=dict(lam=0.25, k=2, gamma=0.5, samples_per_iter=2000, seeds=20, feedback_cap=3000,
                                                       push=_push(0.25, 0.5, 2.5), max_iters=30)),
    "dof5-proof": dict(dof=5, clutter=3, params=dict(lam=0.35, k=2, gamma=0.5, samples_per_iter=2000, seeds=20, feedback_cap=2000,
                                                       push=_push(0.35, 0.5, 2.5), max_iters=30)),
    "dof6-proof": dict(dof=6, clutter=0, params=dict(lam=0.5, k=2, gamma=0.35, samples_per_iter=1000, seeds=20, feedback_cap=2000,
                                                       push=_push(0.5, 0.35, 2.15), max_iters=40, max_edges=200_000_000)),
    # the same arm with three clutter primitives in reach of the distal links (clutter seed 5; seeds 11 and 3 leave the loop
    # with 2-4 free points in a joint-limit corner after 40 iterations)
    "dof6-clutter-proof": dict(dof=6, clutter=3, scene=dict(seed=5),
                               params=dict(lam=0.5, k=2, gamma=0.35, samples_per_iter=1000, seeds=20, feedback_cap=2000,
                                           push=_push(0.5, 0.35, 2.15), max_iters=40, max_edges=200_000_000)),
    # the 3-DoF twin the reference's CPU loop finishes in minutes (its own arm3wall pattern, same generator)
    "dof3-proof": dict(dof=3, clutter=0, params=dict(lam=0.15, k=2, gamma=2.0, samples_per_iter=600, seeds=20, max_iters=30)),
}
