"""Roadmap behaviour, scenario for scenario as the reference tests it (pkg/tests/test_planner.py): growth, labelling,
path queries, free-point insertion, graph invariants.  Every scenario runs twice: with the oracle's collision predicate
injected (CPU suite: pins the batched plan/commit logic) and with the device `batch_check` (GPU suite)."""

from __future__ import annotations

import numpy as np
import pytest

from tests.conftest import oracle_model

START = np.array([0.15, 0.5])
GOAL = np.array([0.85, 0.5])


def _models():
    from paper_2406_04795_b200 import collision as CO
    joints = [CO.Joint("prismatic", (1, 0, 0), CO.Pose.from_xyz_rpy(), (0.0, 1.0)),
              CO.Joint("prismatic", (0, 1, 0), CO.Pose.from_xyz_rpy(), (0.0, 1.0))]
    robot = CO.RobotModel(joints, [CO.LinkSphere(link=2, offset=(0, 0, 0), radius=0.02)])
    box = lambda size, xyz: CO.Box(size, CO.Pose.from_xyz_rpy(xyz=xyz))           # noqa: E731
    scenes = {
        "empty": CO.Scene([]),
        "wall": CO.Scene([box((0.2, 4, 2), (0.5, 0.5, 0))]),        # splits left from right
        "gap": CO.Scene([box((0.2, 0.8, 2), (0.5, 0.6, 0))]),       # free corridor underneath (y < 0.2)
        "blocked": CO.Scene([box((4, 4, 4), (0.5, 0.5, 0))]),
    }
    return robot, scenes


@pytest.fixture(params=["oracle", pytest.param("device", marks=pytest.mark.gpu)])
def make(request):
    """make(scene_name, seed=0, delta=0.05, knn=10) -> Roadmap using the parametrised collision predicate."""
    from paper_2406_04795_b200 import collision as CO, planner as PLN
    robot, scenes = _models()

    def factory(scene_name, seed=0, delta=0.05, knn=10):
        scene = scenes[scene_name]
        check = None
        if request.param == "oracle":
            from oracle import permatrace_oracle as O
            orobot, oscene = oracle_model(CO.robot_to_dict(robot), CO.scene_to_dict(scene))
            check = lambda pts: O.batch_hits(orobot, oscene, np.ascontiguousarray(pts, dtype=np.float64))   # noqa: E731
        return PLN.Roadmap(robot, scene, delta=delta, knn=knn, rng=np.random.default_rng(seed), check=check)

    return factory


def rows_as_set(array) -> set:
    return {row.tobytes() for row in array}


def test_union_find():
    from paper_2406_04795_b200.planner import UnionFind
    uf = UnionFind()
    ids = [uf.add() for _ in range(6)]
    assert ids == list(range(6)) and not uf.same(0, 1)
    uf.union(0, 1); uf.union(2, 3); uf.union(1, 3)
    assert uf.same(0, 2) and uf.same(1, 3) and not uf.same(0, 4)
    uf.union(0, 1); uf.union(3, 0)                                  # idempotent
    assert sorted(uf.find(i) == uf.find(0) for i in range(6)) == [False, False, True, True, True, True]
    assert uf.size[uf.find(0)] == 4


# ---- grow -------------------------------------------------------------------------------------------------------
def test_grow_empty_scene_is_one_component(make):
    from paper_2406_04795_b200.planner import grow, insert_free_points
    rm = make("empty")
    insert_free_points(rm, [START, GOAL])
    assert grow(rm, 100) == 100
    anchor = rm.index_of(START)
    assert all(rm.components.same(anchor, i) for i in range(len(rm)))


def test_grow_blocked_and_walled(make):
    from paper_2406_04795_b200.planner import grow
    rm = make("blocked")
    assert grow(rm, 50) == 0 and len(rm) == 50 and not any(rm.free)
    rm = make("wall")
    added = grow(rm, 120)
    assert added == sum(rm.free) and 0 < added < 120                # the wall swallows some samples
    assert rm.collision_batches == 2                                # samples, then all candidate segments


def test_fixed_seed_reproduces_roadmap(make):
    from paper_2406_04795_b200.planner import grow, insert_free_points
    runs = []
    for _ in range(2):
        rm = make("gap", seed=7)
        insert_free_points(rm, [START, GOAL])
        grow(rm, 80)
        runs.append(rm)
    a, b = runs
    assert len(a) == len(b) and a.free == b.free and a.neighbors == b.neighbors
    assert all(np.array_equal(qa, qb) for qa, qb in zip(a.configs, b.configs))
    assert a.components.parent == b.components.parent


def test_validation(make):
    from paper_2406_04795_b200.planner import Roadmap, grow
    robot, scenes = _models()
    with pytest.raises(ValueError):
        grow(make("empty"), 0)
    with pytest.raises(ValueError):
        Roadmap(robot, scenes["empty"], delta=0.0)
    with pytest.raises(ValueError):
        Roadmap(robot, scenes["empty"], delta=0.05, knn=0)


# ---- labelled samples -----------------------------------------------------------------------------------------------
def test_labels_partition_the_roadmap(make):
    from paper_2406_04795_b200.planner import grow, insert_free_points, labeled_samples
    rm = make("gap")
    insert_free_points(rm, [START, GOAL])
    grow(rm, 60)
    labels = labeled_samples(rm, START)
    assert labels.positive.shape[0] + labels.negative.shape[0] == len(rm)
    assert not rows_as_set(labels.positive) & rows_as_set(labels.negative)
    assert START.tobytes() in rows_as_set(labels.positive)
    rm = make("empty")
    insert_free_points(rm, [START, GOAL])
    grow(rm, 60)
    assert labeled_samples(rm, START).negative.shape[0] == 0       # fully connected: no negatives at all


def test_wall_puts_goal_side_in_negative(make):
    from paper_2406_04795_b200.planner import grow, insert_free_points, labeled_samples
    rm = make("wall")
    insert_free_points(rm, [START, GOAL])
    grow(rm, 150)
    negative = rows_as_set(labeled_samples(rm, START).negative)
    right_side = [q for q in rm.configs if q[0] > 0.65]
    assert right_side and all(q.tobytes() in negative for q in right_side)


def test_isolated_start_and_unknown_anchor(make):
    from paper_2406_04795_b200.planner import insert_free_points, labeled_samples
    rm = make("wall")
    with pytest.raises(KeyError):
        labeled_samples(rm, START)
    insert_free_points(rm, [START])
    rm.add_config((0.5, 0.5), free=False)
    labels = labeled_samples(rm, START)
    assert labels.positive.shape == (1, 2) and np.array_equal(labels.positive[0], START)
    assert labels.negative.shape == (1, 2)


# ---- path queries ---------------------------------------------------------------------------------------------------
def test_find_path(make):
    from paper_2406_04795_b200.planner import find_path, grow, insert_free_points
    rm = make("empty")
    insert_free_points(rm, [START, GOAL])
    grow(rm, 100)
    path = find_path(rm, START, GOAL)
    assert path is not None and np.array_equal(path[0], START) and np.array_equal(path[-1], GOAL)
    assert all(rm.index_of(b) in rm.neighbors[rm.index_of(a)] for a, b in zip(path, path[1:]))
    assert rm.first_blocked_segment(path, rm.delta / 2.0) is None
    rm = make("wall")
    insert_free_points(rm, [START, GOAL])
    grow(rm, 100)
    assert find_path(rm, START, GOAL) is None
    rm = make("empty")
    insert_free_points(rm, [START, GOAL, (0.5, 0.95)])
    assert len(find_path(rm, START, GOAL)) == 2                     # the straight edge beats the detour
    rm = make("empty")
    insert_free_points(rm, [START])
    with pytest.raises(KeyError):
        find_path(rm, START, GOAL)


def test_first_blocked_segment_reports_the_first_failure(make):
    rm = make("wall")
    path = [np.array([0.05, 0.2]), np.array([0.3, 0.2]), np.array([0.7, 0.2]), np.array([0.95, 0.2]), np.array([0.3, 0.9])]
    assert rm.first_blocked_segment(path, rm.delta / 2.0) == 1       # 0.3 -> 0.7 crosses the wall; so does the last one
    assert rm.first_blocked_segment(path[:2], rm.delta) is None
    assert rm.first_blocked_segment(path[:1], rm.delta) is None
    assert not rm.validate_segment(path[1], path[2]) and rm.validate_segment(path[0], path[1])


# ---- free-point insertion ------------------------------------------------------------------------------------------
def test_bridge_merges_components(make):
    from paper_2406_04795_b200.planner import find_path, insert_free_points
    rm = make("gap")
    left, right = np.array([0.15, 0.8]), np.array([0.85, 0.8])
    insert_free_points(rm, [left, right])
    assert not rm.components.same(rm.index_of(left), rm.index_of(right))
    assert insert_free_points(rm, [(0.15, 0.1), (0.5, 0.05), (0.85, 0.1)]) == 3
    assert rm.components.same(rm.index_of(left), rm.index_of(right))
    assert find_path(rm, left, right) is not None


def test_insert_dedup_rules(make):
    from paper_2406_04795_b200.planner import insert_free_points
    rm = make("empty")
    assert insert_free_points(rm, np.empty((0, 2))) == 0 and len(rm) == 0
    assert insert_free_points(rm, [START]) == 1
    assert insert_free_points(rm, [START]) == 0 and len(rm) == 1
    assert insert_free_points(rm, [START + 1e-12]) == 0
    assert insert_free_points(rm, [START + 1e-6]) == 1
    # duplicates INSIDE one call are tested against the points inserted earlier in the same call
    assert insert_free_points(rm, [GOAL, GOAL + 1e-12, GOAL + 1e-3], dedup_tol=1e-9) == 2


# ---- graph invariants -----------------------------------------------------------------------------------------------
def test_graph_invariants(make):
    from paper_2406_04795_b200.planner import grow, insert_free_points
    rm = make("gap", seed=3)
    insert_free_points(rm, [START, GOAL])
    grow(rm, 150)
    edges = [(i, j) for i in range(len(rm)) for j in rm.neighbors[i] if i < j]
    assert edges
    ends_a = np.array([rm.configs[i] for i, _ in edges])
    ends_b = np.array([rm.configs[j] for _, j in edges])
    from paper_2406_04795_b200.planner import _segment_grids
    points, sizes = _segment_grids(ends_a, ends_b, rm.delta / 2.0)
    assert not np.asarray(rm.check(points)).any()                   # every edge survives half-step re-validation
    assert all(rm.free[i] and rm.free[j] for i, j in edges)
    assert all(rm.neighbors[j][i] == w for i in range(len(rm)) for j, w in rm.neighbors[i].items())
    assert all(len(d) == 0 for d, free in zip(rm.neighbors, rm.free) if not free)
    # union-find == connected components of the neighbour graph
    label = list(range(len(rm)))
    for seed in range(len(rm)):
        if label[seed] != seed:
            continue
        stack = [seed]
        while stack:
            node = stack.pop()
            for other in rm.neighbors[node]:
                if label[other] != seed:
                    label[other] = seed
                    stack.append(other)
    for i in range(len(rm)):
        for j in range(i + 1, len(rm)):
            assert rm.components.same(i, j) == (label[i] == label[j])
