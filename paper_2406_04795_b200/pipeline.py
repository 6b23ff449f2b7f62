"""The slice of ``permatrace/pipeline.py`` that sits on the hot path.

Only what `refine` and the benchmark need lives here: `Problem` (pipeline.py:80-107) and the
non-free checker the refinement stage calls (pipeline.py:256-270).  The solve loop, certificates
and their text formats are the *callers* of this path and stay in the
reference package; INTEGRATION.md shows how they bind to this module.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .collision import RobotModel, Scene, _check, config_in_collision, device_checker, joint_limits

__all__ = ["Problem", "not_free_checker", "_not_free_checker"]


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
