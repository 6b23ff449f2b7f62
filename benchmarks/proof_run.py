#!/usr/bin/env python
"""End-to-end infeasibility proof on the fence scenes (scenes.fence_problem_dict): `pipeline.solve` until it returns an
`InfeasibilityProof` that `verify_proof` accepts, with the per-iteration records and the device share of the wall time.

    python benchmarks/proof_run.py --workload dof5-proof
    python benchmarks/proof_run.py --dof 6 --clutter 0 --lam 0.3 --gamma 0.5 --samples 6000 --feedback-cap 4000
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import paper_2406_04795_b200 as P
    from paper_2406_04795_b200 import pipeline as PL, scenes
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default=None)
    ap.add_argument("--dof", type=int, default=5)
    ap.add_argument("--clutter", type=int, default=None)
    ap.add_argument("--lam", type=float, default=None)
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--gamma", type=float, default=None)
    ap.add_argument("--samples", type=int, default=None)
    ap.add_argument("--seeds", type=int, default=None)
    ap.add_argument("--reg", type=float, default=None)
    ap.add_argument("--push-mult", type=float, default=None, help="push = mult * lam * sqrt(2 gamma) (reference default: 1)")
    ap.add_argument("--q1-limit", type=float, default=None)
    ap.add_argument("--limit", type=float, default=None, help="limits of joints 2..n (default 1.2)")
    ap.add_argument("--rng-seed", type=int, default=None)
    ap.add_argument("--scene-seed", type=int, default=None, help="seed of the clutter placement")
    ap.add_argument("--feedback-cap", type=int, default=None)
    ap.add_argument("--max-iters", type=int, default=30)
    ap.add_argument("--timeout", type=float, default=600.0)
    ap.add_argument("--max-edges", type=int, default=200_000_000)
    args = ap.parse_args()
    if args.workload:
        conf = dict(scenes.PROOF_CONFIGS[args.workload])
    else:
        conf = dict(dof=args.dof, clutter=6, params={})
    over = dict(conf.get("params", {}))
    for key, val in (("lam", args.lam), ("k", args.k), ("gamma", args.gamma), ("samples_per_iter", args.samples),
                     ("seeds", args.seeds), ("regularization", args.reg), ("feedback_cap", args.feedback_cap),
                     ("rng_seed", args.rng_seed)):
        if val is not None:
            over[key] = val
    clutter = conf["clutter"] if args.clutter is None else args.clutter
    if args.push_mult is not None:
        over["push"] = args.push_mult * over["lam"] * np.sqrt(2.0 * over["gamma"])
    extra = dict(conf.get("scene", {}))
    if args.q1_limit is not None:
        extra["q1_limit"] = args.q1_limit
    if args.limit is not None:
        extra["limit"] = args.limit
    if args.scene_seed is not None:
        extra["seed"] = args.scene_seed
    pf = PL.problem_file_from_dict(scenes.fence_problem_dict(conf["dof"], clutter=clutter, **extra))
    problem = pf.problem()
    params = PL.SolveParams(**{**dict(max_iters=args.max_iters, timeout=args.timeout, max_edges=args.max_edges), **over})
    t0 = time.perf_counter()
    out = PL.solve(problem, params)
    dt = time.perf_counter() - t0
    stats = out.stats if hasattr(out, "stats") else None
    for rec in (stats.iterations if stats else []):
        print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in rec.items()}), flush=True)
    line = {"workload": args.workload or f"dof{conf['dof']}", "clutter": clutter, "params": over, "outcome": type(out).__name__,
            "seconds": dt, "iterations": len(stats.iterations) if stats else None}
    if isinstance(out, PL.InfeasibilityProof):
        t1 = time.perf_counter()
        rep = PL.verify_proof(out, problem)
        line.update(verified=rep.ok, verify_s=time.perf_counter() - t1, points=int(out.points.shape[0]),
                    coarse_edges=out.coarse_edges, coarse_cells=out.coarse_cells, support=int(out.manifold.support.shape[0]),
                    free_points=0,
                    device_s=sum(r.get("trace_s", 0) + r.get("refine_s", 0) + r.get("train_s", 0) for r in stats.iterations))
    elif hasattr(out, "reason"):
        line["reason"] = out.reason
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
