"""The smoke() case: one small invocation of the whole hot path on cuda:0, checked against the
CPU oracle on the same inputs (3-DoF learned manifold, 2-fold refinement, arm + 3 obstacles)."""

from __future__ import annotations

import numpy as np


def run_smoke(verbose: bool = True):
    import paper_2406_04795_b200 as P
    from paper_2406_04795_b200 import collision as CO
    from paper_2406_04795_b200.scenes import arm_robot_dict, arm_scene_dict
    from oracle import permatrace_oracle as O
    from tests.conftest import Golden, oracle_model, trace_inputs

    g = Golden("traces")
    tag, n = "kclf_n3", 3
    inp = trace_inputs(g, tag)
    gbb, bar = g[f"{tag}_gbb"], g[f"{tag}_barrier"]
    barrier = P.BoxBarrier(bar[2:2 + n], bar[2 + n:], bar[0], bar[1])
    manifold = P.KernelClassifierManifold(g[f"{tag}_support"], g[f"{tag}_weights"], gbb[0], gbb[1], barrier=barrier)
    cfg = P.TraceConfig(P.LatticeConfig(n, inp["scale"], inp["offset"]), box=inp["box"], eps=inp["eps"])
    result = P.trace(inp["seeds"], manifold, cfg)
    cells = P.coarse_cells(result)
    rd, sd = arm_robot_dict(n), arm_scene_dict(3)

    class Prob:
        robot, scene = CO.robot_from_dict(rd), CO.scene_from_dict(sd)

    refined = P.refine(cells, P.build_template(n, 2), manifold, P.not_free_checker(Prob), cfg)

    field = O.Field.rbf(g[f"{tag}_support"], g[f"{tag}_weights"], gbb[0], gbb[1],
                        barrier=(bar[0], bar[1], bar[2:2 + n], bar[2 + n:]))
    ot = O.Trace(field, n, inp["scale"], inp["offset"], inp["box"], inp["max_edges"], inp["eps"]).run(inp["seeds"])
    base, mask, _ = result.edges.arrays()
    want_base = np.array([e[0] for e in ot.edges])
    want_mask = np.array([sum(1 << l for l in e[1][0]) for e in ot.edges])
    assert np.array_equal(base, want_base) and np.array_equal(mask, want_mask), "traced edge list differs from the oracle"
    assert result.closure_ok == ot.closure_ok
    assert np.allclose(result.points, ot.points(), rtol=1e-5, atol=1e-9)
    ocells = O.coarse_cells(ot.edges)
    robot, scene = oracle_model(rd, sd)
    oref = O.refine(ocells, O.build_template(n, 2), field, lambda p: O.not_free(robot, scene, p),
                    inp["scale"], inp["offset"], 2, inp["eps"])
    assert refined.points.shape == oref["points"].shape, (refined.points.shape, oref["points"].shape)
    assert np.allclose(refined.points, oref["points"], rtol=1e-5, atol=1e-9)
    assert np.array_equal(refined.in_collision, oref["in_collision"])
    if verbose:
        print(f"smoke: {len(result.edges)} edges, {len(cells)} cells, {refined.points.shape[0]} points, "
              f"{int((~refined.in_collision).sum())} free -- identical to the CPU oracle")
