"""Overhead of the multi-GPU driver itself: ShardedProof with a process group of ONE rank (no data crosses any link)
against the single-GPU device pipeline on the same workload, over the NCCL backend.  What differs is the orchestration: per-wave candidate
records and winner ranking through torch tensors, candidates merged by all_gather, dedup + labels as separate calls.

    python benchmarks/sharded_overhead.py [workload]
"""
import os
import sys
import time
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from bench import build_workload  # noqa: E402
import paper_2406_04795_b200 as P  # noqa: E402
from paper_2406_04795_b200 import engine  # noqa: E402
from paper_2406_04795_b200.distributed import CudaEngine, ShardedProof  # noqa: E402


def timed(fn, reps=5):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t0) / reps


def main():
    wl = build_workload(sys.argv[1] if len(sys.argv) > 1 else "dof6")
    checker = P.not_free_checker(wl.problem)
    seeds = torch.from_numpy(wl.arrays.seeds).cuda()
    pipe = engine.DevicePipeline(wl.manifold, wl.cfg, wl.template, checker)
    single = timed(lambda: pipe.step(seeds.data_ptr(), seeds.shape[0]))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29541")
    # the real transport: a one-rank NCCL group (NCCL refuses two ranks on one device)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    proof = ShardedProof(CudaEngine(wl.manifold, wl.cfg, wl.template, checker), gather_result=False)
    sharded = timed(lambda: proof.run(seeds))
    # ... and the same with every collective of the fully sharded path actually issued to NCCL (count matrix, record
    # all_to_all and winner all_gather per wave, sample sort, ghost exchange, pin rounds): their launch + host-sync cost
    os.environ["PERMATRACE_B200_FORCE_COLLECTIVES"] = "1"
    forced_proof = ShardedProof(CudaEngine(wl.manifold, wl.cfg, wl.template, checker), gather_result=False)
    res = forced_proof.run(seeds)
    forced = timed(lambda: forced_proof.run(seeds))
    print(f"device pipeline {single:.2f} ms | ShardedProof(world=1, replicated path) {sharded:.2f} ms | "
          f"fully sharded path, all collectives through NCCL on one rank {forced:.2f} ms "
          f"(levels {res['levels']}, pin rounds {res.get('pin_rounds')}, points {res['points_total']})")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
