cd /root/repo
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "taylor or full_size_refine or ill_conditioned or large_support or bisection or tc_" 2>&1 | tail -3
for w in dof6 dof6-s4096 dof5; do python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2_f_$w.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/r2_f_$w.json')); k=d['kernels']; print('$w', round(d['ms_per_step'],2), d['config'].get('rows_left_to_evaluation_kernels'), d['roofline']['frac'], [(n, round(v['ms'],2)) for n,v in sorted(k.items(), key=lambda kv:-kv[1]['ms'])[:5]])"; done
