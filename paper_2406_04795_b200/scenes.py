"""Synthetic 3/4/5/6-DoF manipulator scenes in the reference's dict/YAML schema.

The reference ships only 2-DoF point robots and the 3-DoF ``arm3wall`` (permatrace/scenes/*.yaml);
BASELINE.json's configs 2-5 need 4/5/6-DoF arms.  These follow the arm3wall pattern extended
(SURVEY.md section 8d): a serial chain of revolute joints alternating z / y axes, link length 0.4,
four collision spheres of radius 0.06 per link, box / cylinder / sphere obstacles.  The dicts load
through ``collision.robot_from_dict`` / ``scene_from_dict`` here and in the reference alike.
"""

from __future__ import annotations

import numpy as np

__all__ = ["arm_robot_dict", "arm_scene_dict", "synthetic_support", "BENCH_CONFIGS"]


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
    # support set of the size the reference's own solve loop ends with (arm3wall: 4 199 roadmap samples)
    "dof6-s4096": dict(n=6, support=4096, lam=0.35, r_split=1.3, obstacles=8),
    # the support-set size the SURVEY expects for real 6-DoF proofs (10^3..10^4 roadmap samples): 8 support chunks
    "dof6-s16384": dict(n=6, support=16384, lam=0.35, r_split=1.3, obstacles=8),
}
