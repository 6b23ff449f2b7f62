cd /root/repo
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 | cut -c1-300
python benchmarks/bfs_scaling.py --dim 6 --lambdas 0.14 0.1 --reps 2 > gpurun_out/r2_bfs_scaling_v2.jsonl 2>/dev/null; cut -c1-900 gpurun_out/r2_bfs_scaling_v2.jsonl
python benchmarks/bfs_scaling.py --dim 4 --lambdas 0.02 --reps 2 2>/dev/null | cut -c1-600
python bench.py --workload dof6 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2_i_dof6.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/r2_i_dof6.json')); print('dof6', round(d['ms_per_step'],2), d['roofline_hbm'])"
