"""Where the time of an end-to-end `solve()` goes: runs the product on the reference's
bundled scenes frozen in tests/golden/solve.npz and prints the per-iteration record next to the reference's wall
time for the same scene (measured when the fixture was generated, Cython backend, this container's CPU).

    python benchmarks/solve_breakdown.py [wall2d|gap2d|arm3wall ...]
"""

from __future__ import annotations

import cProfile
import json
import pstats
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))

from paper_2406_04795_b200 import collision as CO, pipeline as PL  # noqa: E402


def main():
    g = np.load(REPO / "tests" / "golden" / "solve.npz")
    names = [a for a in sys.argv[1:] if not a.startswith("-")] or ["wall2d", "gap2d", "arm3wall"]
    profile = "--profile" in sys.argv
    for name in names:
        rs = json.loads(str(g[f"{name}/robot_scene_json"][0]))
        pf = PL.ProblemFile(CO.robot_from_dict(rs["robot"]), CO.scene_from_dict(rs["scene"]), g[f"{name}/start"],
                            g[f"{name}/goal"], json.loads(str(g[f"{name}/params_json"][0])))
        problem = pf.problem()
        for rep in range(2):                       # the first run pays context creation and template construction
            prof = cProfile.Profile() if profile and rep == 1 else None
            t0 = time.perf_counter()
            if prof:
                prof.enable()
            outcome = PL.solve(problem, pf.solve_params(timeout=600.0))
            if prof:
                prof.disable()
            dt = time.perf_counter() - t0
        stats = outcome.stats
        print(f"{name}: {type(outcome).__name__} in {dt:.3f} s (reference: {float(g[f'{name}/seconds'][0]):.1f} s), "
              f"{len(stats.iterations)} iterations")
        for r in stats.iterations:
            keys = ("roadmap", "positive", "negative", "train_s", "trace_s", "edges", "cells", "refine_s", "points", "free_points")
            print("   ", {k: (round(r[k], 4) if isinstance(r[k], float) else r[k]) for k in keys if k in r}, r.get("skip", ""))
        staged = sum(r.get(k, 0.0) for r in stats.iterations for k in ("train_s", "trace_s", "refine_s"))
        print(f"    train+trace+refine {staged:.3f} s, everything else (roadmap, seeds, verification) {dt - staged:.3f} s")
        if prof:
            pstats.Stats(prof).sort_stats("cumulative").print_stats(18)


if __name__ == "__main__":
    main()
