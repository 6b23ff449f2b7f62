cd /root/repo
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "taylor or full_size_refine or ill_conditioned or large_support or bisection or trace_matches" -s 2>&1 | grep -v "^$" | tail -30 > gpurun_out/r2_taylor_test3.log; cat gpurun_out/r2_taylor_test3.log
for w in dof6 dof6-s4096 dof6-s16384 dof5 dof4; do python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2_e_$w.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/r2_e_$w.json')); k=d['kernels']; print('$w', round(d['ms_per_step'],2), d['config'].get('rows_left_to_evaluation_kernels'), d['roofline']['frac'], [(n, round(v['ms'],2)) for n,v in sorted(k.items(), key=lambda kv:-kv[1]['ms'])[:9]])"; done
python bench.py --workload dof6-proof --steps 1 --warmup 0 > gpurun_out/r2_e_dof6-proof.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/r2_e_dof6-proof.json')); print('dof6-proof', d['value'], d['config']['verified'], d['config']['iterations'], d['device_share'], d['clocks'].get('hbm_used_max_gb'))"
