"""CPU-only tests of the product's host side: the C ABI surface, the host-executable mirrors of the
device lattice arithmetic (same inline functions the kernels compile), the Python value types, and
the loud failure when no GPU is present.  No compute call needs a device here."""

from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from tests.conftest import REPO, mask_of, parts_of_mask

import paper_2406_04795_b200 as P
from paper_2406_04795_b200 import _cabi, lattice as L, subdivision as S, manifold as M, collision as CO, tracer as T


# ---- C ABI -------------------------------------------------------------------------------------
def test_every_declared_symbol_is_exported():
    header = (REPO / "include" / "permatrace_b200.h").read_text()
    declared = set(re.findall(r"\b(pt_[a-z0-9_]+)\s*\(", header))
    declared -= {"pt_trace_stats", "pt_refine_stats"}
    assert declared, "header parse failed"
    for name in sorted(declared):
        assert hasattr(_cabi.lib, name), f"{name} declared in include/permatrace_b200.h but not exported"
    assert declared == set(_cabi.DECLARED_SYMBOLS)
    assert _cabi.lib.pt_version() >= 100


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "-lelf", str(_cabi.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError, match="no CPU path|CUDA"):
        M.SphereManifold(np.zeros(3), 1.0).values(np.zeros((2, 3)))
    with pytest.raises(RuntimeError):
        P.backend.rbf_values(np.zeros((1, 2)), np.zeros((1, 2)), np.zeros(1), 1.0, 0.0)



def test_reference_arm_never_maps_the_product_library():
    """`bench.py --impl reference` builds its workload and runs the CPU sample without importing the product package or
    mapping libpermatrace_b200.so (the driver watches which .so files each arm loads)."""
    import subprocess
    import sys
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import bench\n"
        "bench.CPU_RUNS, bench.CPU_RUN_LEN = 2, 3\n"
        "info = bench.cpu_sample('dof3', 2, max_edges=60, runs=2, run_len=3, prefer_reference=False)\n"
        "assert info['kind'] == 'port' and info['coarse_edges'] == 60 and info['cells_refined'] == 6\n"
        "maps = open('/proc/self/maps').read()\n"
        "assert 'libpermatrace_b200' not in maps, 'product library mapped by the reference arm'\n"
        "assert not any(m.startswith('paper_2406_04795_b200') for m in sys.modules), 'product package imported'\n"
        "print('clean')\n" % str(REPO))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "clean" in out.stdout, out.stderr[-2000:]


def test_product_never_imports_the_oracle():
    for path in (REPO / "paper_2406_04795_b200").rglob("*"):
        if path.suffix in (".py", ".cu", ".cuh", ".h", ".sh") and path.is_file():
            text = path.read_text()
            assert "permatrace_oracle" not in text and "liboracle" not in text, path
            assert not re.search(r"^\s*(from|import)\s+oracle\b", text, re.M), path


# ---- device lattice arithmetic, executed on the host ------------------------------------------------
@pytest.mark.parametrize("n", [2, 3, 4, 5, 6])
def test_device_coface_arithmetic_matches_reference_plans(golden, n):
    rows = golden("lattice")[f"plan_n{n}"]
    at = 0
    buf = np.zeros((256, 10), dtype=np.int32)

    def vec(plus, minus):
        return [((plus >> d) & 1) - ((minus >> d) & 1) for d in range(n)]

    for mask in range(1, 1 << n):
        nc = _cabi.lib.pt_host_expansion_plan(n, mask, buf.ctypes.data, 256)
        assert nc == (2 ** bin(mask).count("1") - 2) + (2 ** (n + 1 - bin(mask).count("1")) - 2)
        for j in range(nc):
            r = buf[j]
            got = [mask, j, *vec(r[0], r[1]), *vec(r[2], r[3]), int(r[4]), int(r[5]), *vec(r[6], r[7]), int(r[8]), int(r[9])]
            assert got == list(rows[at]), (n, mask, j)
            at += 1
    assert at == rows.shape[0]


@pytest.mark.parametrize("n", [2, 3, 4, 5, 6])
def test_device_cellcoface_arithmetic_matches_reference(golden, n):
    rows = golden("lattice")[f"cellcofaces_n{n}"]
    buf = np.zeros((720, 1 + n), dtype=np.int32)
    for mask in sorted(set(int(m) for m in rows[:, 0])):
        want = {tuple(int(v) for v in r[1:]) for r in rows[rows[:, 0] == mask]}
        nc = _cabi.lib.pt_host_cellcofaces(n, mask, buf.ctypes.data, 720)
        got = set()
        for t in range(nc):
            y = int(buf[t, 0])
            base = tuple(-((y >> d) & 1) for d in range(n))
            got.add(base + tuple(int(v) for v in buf[t, 1:]))
        assert nc == len(want) and got == want, (n, mask)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 7])
def test_perm_rank_roundtrip_is_lexicographic(n):
    from itertools import permutations
    perm = np.zeros(n, dtype=np.uint8)
    for rank, p in enumerate(permutations(range(n))):
        if rank > 400:
            break
        arr = np.asarray(p, dtype=np.uint8)
        assert _cabi.lib.pt_host_perm_rank(n, arr.ctypes.data) == rank
        assert _cabi.lib.pt_host_perm_unrank(n, rank, perm.ctypes.data) == 0
        assert tuple(perm) == p


# ---- Python value types ---------------------------------------------------------------------------
def _ref_like(simplex):
    return (tuple(simplex.base), tuple(simplex.parts))


@pytest.mark.parametrize("n", [2, 3, 4, 5, 6])
def test_host_lattice_functions_match_reference(golden, n):
    from oracle import permatrace_oracle as O
    rng = np.random.default_rng(n)
    for mask in range(1, 1 << n):
        base = tuple(int(v) for v in rng.integers(-3, 4, size=n))
        edge = L.PermSimplex(base, parts_of_mask(mask, n))
        assert [_ref_like(f) for f in L.cofaces2_of_edge(edge)] == O.cofaces2_of_edge(_ref_like(edge))
        if n <= 4:
            assert [_ref_like(c) for c in L.cellcofaces_of_edge(edge)] == O.cellcofaces_of_edge(_ref_like(edge))
        tri = L.cofaces2_of_edge(edge)[0]
        assert [_ref_like(e) for e in L.edges_of_2simplex(tri)] == O.pair_edges(_ref_like(tri))
        # canonicalize is idempotent and rotation-invariant
        for rot in range(3):
            verts = L.simplex_vertices(tri)
            rotated = L.PermSimplex(verts[rot], tri.parts[rot:] + tri.parts[:rot])
            assert L.canonicalize(rotated) == tri
    g = golden("lattice")
    cell = L.PermSimplex((0, 0, 0), ((2,), (0,), (1,), (3,)))
    b, m = L.edges_to_arrays(L.edges_of_cell(cell), 3)
    assert np.array_equal(b, g["fig2_cell_edges_base"]) and np.array_equal(m, g["fig2_cell_edges_mask"])


@pytest.mark.parametrize("n", [2, 3, 5])
def test_host_locate_point(golden, n):
    g = golden("lattice")
    cfg = L.LatticeConfig(n, 0.37, tuple(0.05 * (i + 1) for i in range(n)))
    cells = [L.locate_point(p, cfg) for p in g[f"locate_n{n}_points"]]
    b, p = L.cells_to_arrays(cells, n)
    assert np.array_equal(b, g[f"locate_n{n}_base"]) and np.array_equal(p, g[f"locate_n{n}_perm"])
    assert L.cells_from_arrays(b, p) == cells


def test_lattice_validation():
    with pytest.raises(ValueError):
        L.LatticeConfig(1)
    with pytest.raises(ValueError):
        L.LatticeConfig(3, 0.0)
    with pytest.raises(ValueError):
        L.LatticeConfig(3, 1.0, (0.0, 0.0))
    with pytest.raises(ValueError):
        L.PermSimplex((0, 0), ((0,), (1,))).validate()
    with pytest.raises(ValueError):
        L.PermSimplex((0, 0), ((1, 0), (2,))).validate()
    L.PermSimplex((0, 0), ((0, 1), (2,))).validate()
    with pytest.raises(ValueError):
        L.locate_point([0.0, np.inf], L.LatticeConfig(2))
    with pytest.raises(ValueError):
        L.edges_of_cell(L.PermSimplex((0, 0), ((0, 1), (2,))))


@pytest.mark.parametrize("n,k", [(2, 2), (3, 3), (5, 2), (6, 2), (4, 4)])
def test_build_template_matches_reference(golden, n, k):
    g = golden("refine")
    t = S.build_template(n, k)
    assert np.array_equal(t.vertices, g[f"template_n{n}_k{k}_v"])
    assert np.array_equal(t.edges, g[f"template_n{n}_k{k}_e"])
    assert np.allclose(t.weights.sum(axis=1), 1.0)
    from math import comb
    assert t.vertices.shape[0] == comb(n + k, k)


def test_template_known_counts():
    t = S.build_template(2, 2)
    assert t.vertices.shape == (6, 2) and t.edges.shape == (9, 2)     # pkg/tests/test_subdivision.py:74-78
    assert S.build_template(6, 2).edges.shape[0] == 182 and S.build_template(6, 3).vertices.shape[0] == 84
    with pytest.raises(ValueError):
        S.build_template(1, 2)
    with pytest.raises(ValueError):
        S.build_template(3, 0)


def test_plan_batches_and_budget():
    t = S.build_template(3, 2)
    per = S._cell_bytes(t)
    assert per == 8 * (10 * 4 + 25 * 8)
    cells = [L.PermSimplex((i, 0, 0), ((0,), (1,), (2,), (3,))) for i in range(10)]
    plan = S.plan_batches(cells, t, 3 * per + 5)
    assert [len(b) for b in plan.batches] == [3, 3, 3, 1] and plan.bytes_per_cell == per
    with pytest.raises(S.BudgetError):
        S.plan_batches(cells, t, per - 1)
    assert S.containment_check((2, 1, 0), 2) and not S.containment_check((1, 2, 0), 2) and not S.containment_check((3, 0, 0), 2)
    assert np.allclose(S.barycentric_weights((2, 1, 0), 2), [0.0, 0.5, 0.5, 0.0])


def test_config_validation_and_text_formats(tmp_path):
    with pytest.raises(ValueError):
        T.TraceConfig(L.LatticeConfig(2), max_edges=0)
    with pytest.raises(ValueError):
        T.TraceConfig(L.LatticeConfig(2), eps=0.0)
    pts = np.array([[0.1, 1 / 3], [2.5, -7e-9]])
    T.write_edgemesh(tmp_path / "m.txt", 2, pts, [(0, 1)])
    dim, back, pairs = T.read_edgemesh(tmp_path / "m.txt")
    assert dim == 2 and np.array_equal(back, pts) and pairs == [(0, 1)]
    with pytest.raises(ValueError):
        T.read_edgemesh(__import__("io").StringIO("EDGEMESH n 2 V 1\n"))
    bar = M.BoxBarrier([-1, -1], [1, 1], 0.125, 4.0)
    m = M.KernelClassifierManifold(np.array([[0.1, 0.2], [0.3, -0.4]]), np.array([1.5, -2.5]), 2.0, 0.25, barrier=bar)
    m2 = M.classifier_from_text(M.classifier_to_text(m))
    assert np.array_equal(m2.support, m.support) and np.array_equal(m2.weights, m.weights)
    assert (m2.gamma, m2.bias, m2.barrier.scale, m2.barrier.gain) == (2.0, 0.25, 0.125, 4.0)
    with pytest.raises(ValueError):
        M.classifier_from_text("KCLF v2\n")
    with pytest.raises(ValueError):
        M.KernelClassifierManifold(np.zeros((2, 2)), np.array([1.0, 2.0]), 1.0)   # one-signed weights, no barrier
    assert isinstance(M.parse_manifold("sphere:r=0.8", 4), M.SphereManifold)
    assert np.array_equal(M.parse_manifold("plane:n=1|0,d=0.25", 2).normal, [1.0, 0.0])
    with pytest.raises(ValueError):
        M.parse_manifold("torus:r=1", 3)


def test_collision_schema_roundtrip_and_validation():
    from paper_2406_04795_b200.scenes import arm_robot_dict, arm_scene_dict
    robot = CO.robot_from_dict(arm_robot_dict(4))
    scene = CO.scene_from_dict(arm_scene_dict(8))
    assert robot.dof == 4 and len(robot.spheres) == 16 and len(scene.obstacles) == 8
    again = CO.robot_from_dict(CO.robot_to_dict(robot))
    assert [j.axis for j in again.joints] == [j.axis for j in robot.joints]
    assert {type(o).__name__ for o in scene.obstacles} == {"Box", "Cylinder", "SphereObstacle"}
    again_scene = CO.scene_from_dict(CO.scene_to_dict(scene))
    assert np.allclose(again_scene.obstacles[0].pose.rotation, scene.obstacles[0].pose.rotation)
    with pytest.raises(ValueError):
        CO.robot_from_dict({"joints": []})
    with pytest.raises(ValueError):
        CO.Joint("screw", (0, 0, 1), CO.Pose(), (-1, 1))
    with pytest.raises(ValueError):
        CO.Box((1, -1, 1), CO.Pose())
    with pytest.raises(ValueError):
        CO.Pose(np.diag([1.0, 1.0, -1.0]))
    with pytest.raises(ValueError):
        CO.batch_check(np.zeros((1, 4)), robot, scene, on_limit="maybe")
    lo, hi = CO.joint_limits(robot)
    assert np.all(lo == -1.5) and np.all(hi == 1.5)


def test_proof_workloads_are_well_formed_problem_files():
    """Every end-to-end proof workload (scenes.PROOF_CONFIGS) is a problem file in the reference's schema: robot and scene
    parse, start / goal have the robot's dimension and respect its limits, the SolveParams overrides are accepted, and the
    bias push stays below 1 (labels are +-1: a larger push cannot separate start from goal)."""
    from paper_2406_04795_b200 import collision as CO, pipeline as PL, scenes
    for name, conf in scenes.PROOF_CONFIGS.items():
        pdict = scenes.fence_problem_dict(conf["dof"], clutter=conf["clutter"], **conf.get("scene", {}))
        robot, scene = CO.robot_from_dict(pdict["robot"]), CO.scene_from_dict(pdict["scene"])
        assert robot.dof == conf["dof"] and len(scene.obstacles) == 1 + conf["clutter"], name
        lo, hi = CO.joint_limits(robot)
        for key in ("start", "goal"):
            q = np.asarray(pdict["problem"][key], dtype=np.float64)
            assert q.shape == (conf["dof"],) and np.all(q >= lo) and np.all(q <= hi), (name, key)
        params = PL.SolveParams(**conf["params"])
        push = params.push if params.push is not None else params.lam * np.sqrt(2.0 * params.gamma)
        assert 0.0 < push < 1.0, name
        # the same dict is what the reference's loader takes (round trip through its YAML-level schema)
        assert set(pdict) == {"robot", "scene", "problem"}
