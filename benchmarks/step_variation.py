import sys, time
sys.path.insert(0, "/root/repo")
import torch
from bench import build_workload
import paper_2406_04795_b200 as P
from paper_2406_04795_b200 import engine
wl = build_workload("dof6"); a = wl.arrays
pipe = engine.DevicePipeline(wl.manifold, wl.cfg, wl.template, P.not_free_checker(wl.problem))
seeds = torch.from_numpy(a.seeds).cuda()
for _ in range(3): pipe.step(seeds.data_ptr(), a.seeds.shape[0])
torch.cuda.synchronize()
ts = []
for _ in range(30):
    t0 = time.perf_counter(); pipe.step(seeds.data_ptr(), a.seeds.shape[0]); torch.cuda.synchronize(); ts.append(1e3 * (time.perf_counter() - t0))
print([round(t, 1) for t in ts])
import os; print(os.cpu_count(), os.getloadavg())
