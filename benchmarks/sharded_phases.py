"""Wall-clock phases of the fully sharded driver (distributed.ShardedProof._run_sharded) on a one-rank NCCL group with
every collective issued (PERMATRACE_B200_FORCE_COLLECTIVES=1): where the orchestration cost of the multi-GPU path sits.

    python benchmarks/sharded_phases.py [workload]
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
from paper_2406_04795_b200 import distributed as D  # noqa: E402


def main():
    wl = build_workload(sys.argv[1] if len(sys.argv) > 1 else "dof6")
    checker = P.not_free_checker(wl.problem)
    seeds = torch.from_numpy(wl.arrays.seeds).cuda()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29543")
    os.environ["PERMATRACE_B200_FORCE_COLLECTIVES"] = "1"
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    eng = D.CudaEngine(wl.manifold, wl.cfg, wl.template, checker)
    proof = D.ShardedProof(eng, gather_result=False)
    marks = []

    def wrap(obj, name, label=None):
        fn = getattr(obj, name)

        def timed(*a, **k):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out = fn(*a, **k)
            torch.cuda.synchronize()
            marks.append((label or name, 1e3 * (time.perf_counter() - t0)))
            return out
        setattr(obj, name, timed)

    for name in ("local_points", "local_cell_keys", "set_cells_from_keys", "candidates", "label", "dedup_mask",
                 "trace_locate", "wave_candidates", "wave_admit", "wave_commit"):
        if hasattr(eng, name):
            wrap(eng, name, "engine." + name)
    for name in ("_range_partition", "_sharded_dedup"):
        wrap(proof, name)
    for cls, names in ((D.ShardedTrace, ("_wave_exchange", "_wave_rank", "run")), (D._Transport, ("_sum", "_gather_rows", "_exchange_rows", "_exchange_counts", "_gather_var"))):
        for name in names:
            fn = getattr(cls, name)

            def make(fn, label):
                def timed(self, *a, **k):
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    out = fn(self, *a, **k)
                    torch.cuda.synchronize()
                    marks.append((label, 1e3 * (time.perf_counter() - t0)))
                    return out
                return timed
            setattr(cls, name, make(fn, f"{cls.__name__}.{name}"))
    for rep in range(4):
        marks.clear()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        proof.run(seeds)
        torch.cuda.synchronize()
        total = 1e3 * (time.perf_counter() - t0)
    agg = {}
    for k, v in marks:
        a = agg.setdefault(k, [0, 0.0]); a[0] += 1; a[1] += v
    print(f"total {total:.2f} ms")
    for k, (c, v) in agg.items():
        print(f"  {k:32s} x{c:3d} {v:8.2f} ms")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
