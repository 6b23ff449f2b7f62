"""Shared fixtures.  `-m "not gpu"` covers the oracle against the reference's golden vectors, host
logic and the C-ABI surface; `-m gpu` holds the parity tests proper (CUDA path vs oracle/golden)."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parent.parent
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))

GOLDEN = REPO / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Make sure the oracle's C kernels and the CUDA library exist (compiles only, no GPU needed)."""
    import shutil
    import subprocess
    import __graft_entry__ as entry
    lib = REPO / "paper_2406_04795_b200" / "libpermatrace_b200.so"
    if shutil.which("nvcc") is None and lib.exists():
        # no CUDA toolkit on this machine but a built library travelled with the tree: only the oracle needs compiling
        subprocess.run(["make", "-s", "-C", str(REPO / "oracle")], check=True)
        return
    entry.build()


class Golden:
    def __init__(self, name):
        self.z = np.load(GOLDEN / f"{name}.npz")

    def __getitem__(self, key):
        return self.z[key]

    def __contains__(self, key):
        return key in self.z.files


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = Golden(name)
        return cache[name]

    return load


# ---- helpers shared by oracle and GPU tests --------------------------------------------------------

def parts_of_mask(mask, n):
    p1 = tuple(d for d in range(n) if mask >> d & 1)
    p2 = tuple(d for d in range(n) if not mask >> d & 1) + (n,)
    return (p1, p2)


def mask_of(part):
    m = 0
    for label in part:
        m |= 1 << label
    return m


def trace_inputs(g, tag):
    lat = g[f"{tag}_lattice"]
    n = int(lat[0])
    box = g[f"{tag}_box"] if f"{tag}_box" in g else None
    cfgv = g[f"{tag}_cfg"]
    return dict(n=n, scale=float(lat[1]), offset=tuple(float(v) for v in lat[2:2 + n]),
                box=None if box is None else (tuple(box[0]), tuple(box[1])),
                max_edges=int(cfgv[0]), eps=float(cfgv[1]), seeds=g[f"{tag}_seeds"])


def analytic_spec(tag):
    """(kind, args) of the analytic golden traces (see make_golden.py)."""
    if tag.startswith("sphere_n"):
        n = int(tag.split("_")[1][1:])
        return "sphere", (np.zeros(n), 0.8)
    return {
        "ellipsoid_box": ("ellipsoid", ([0.1, -0.2, 0.05], [0.9, 0.6, 0.7])),
        "sphere_cap": ("sphere", (np.zeros(3), 0.8)),
        "plane_box": ("plane", ([1.0, 0.5, -0.25], 0.1)),
    }[tag]


ANALYTIC_TRACES = ["sphere_n2", "sphere_n3", "sphere_n4", "sphere_n5", "ellipsoid_box", "sphere_cap", "plane_box"]
LEARNED_TRACES = ["kclf_n3", "kclf_n4", "kclf_n5", "kclf_n6"]


def robot_scene_dicts(n, nobs, seed=7):
    from paper_2406_04795_b200.scenes import arm_robot_dict, arm_scene_dict
    return arm_robot_dict(n), arm_scene_dict(nobs, seed)


PRISM_ROBOT = {
    "joints": [
        {"type": "prismatic", "axis": [1, 0, 0], "origin": {"xyz": [0, 0, 0.1], "rpy": [0.1, 0.2, 0.3]}, "limits": [-1, 1]},
        {"type": "revolute", "axis": [0, 1, 1], "origin": {"xyz": [0.3, 0, 0], "rpy": [0, 0, 0]}, "limits": [-2, 2]},
    ],
    "spheres": [{"link": 0, "offset": [0, 0, 0], "radius": 0.1}, {"link": 2, "offset": [0.2, 0.1, 0], "radius": 0.05},
                {"link": 1, "offset": [0.1, 0, 0], "radius": 0.07}],
}
PRISM_SCENE = {"obstacles": [
    {"type": "cylinder", "height": 0.5, "radius": 0.2, "origin": {"xyz": [0.6, 0.1, 0.0], "rpy": [0.5, 0.1, 0.0]}},
    {"type": "sphere", "radius": 0.25, "origin": {"xyz": [-0.7, 0.0, 0.2]}},
    {"type": "box", "size": [0.3, 0.2, 0.4], "origin": {"xyz": [0.1, 0.6, 0.0], "rpy": [0, 0, 0.7]}}]}


def oracle_model(robot_dict, scene_dict):
    """Reference-schema dicts -> the oracle's plain dict model (uses only numpy)."""
    def rpy(r):
        r, p, y = (float(v) for v in r)
        cr, sr, cp, sp, cy, sy = np.cos(r), np.sin(r), np.cos(p), np.sin(p), np.cos(y), np.sin(y)
        rx = np.array([[1, 0, 0], [0, cr, -sr], [0, sr, cr]])
        ry = np.array([[cp, 0, sp], [0, 1, 0], [-sp, 0, cp]])
        rz = np.array([[cy, -sy, 0], [sy, cy, 0], [0, 0, 1]])
        return rz @ ry @ rx

    def pose(o):
        o = o or {}
        if "rotation" in o:                     # canonical form written by robot_to_dict / scene_to_dict
            return np.asarray(o["rotation"], dtype=np.float64), np.asarray(o["translation"], dtype=np.float64)
        return rpy(o.get("rpy", (0, 0, 0))), np.asarray(o.get("xyz", (0, 0, 0)), dtype=np.float64)

    joints = []
    for j in robot_dict["joints"]:
        rot, trans = pose(j.get("origin"))
        axis = np.asarray(j["axis"], dtype=np.float64)
        joints.append(dict(kind=j["type"], axis=tuple(axis / np.linalg.norm(axis)), rot=rot, trans=trans,
                           limits=tuple(float(v) for v in j["limits"])))
    spheres = [dict(link=int(s["link"]), offset=tuple(float(v) for v in s["offset"]), radius=float(s["radius"]))
               for s in robot_dict["spheres"]]
    scene = []
    for o in scene_dict["obstacles"]:
        rot, trans = pose(o.get("origin"))
        if o["type"] == "box":
            dims = tuple(float(v) for v in o["size"])
        elif o["type"] == "cylinder":
            dims = (float(o["height"]), float(o["radius"]), 0.0)
        else:
            dims = (float(o["radius"]), 0.0, 0.0)
        scene.append(dict(type=o["type"], rot=rot, trans=trans, dims=dims))
    return dict(joints=joints, spheres=spheres), scene
