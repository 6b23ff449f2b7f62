cd /root/repo
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 | cut -c1-300
for w in dof6 dof6-stress dof6-s16384; do python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2_h_$w.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/r2_h_$w.json')); k=d['kernels']; print('$w', round(d['ms_per_step'],2), d['config'].get('rows_left_to_evaluation_kernels'), d['config']['points_checked'], d['roofline']['frac'], [(n, round(v['ms'],2)) for n,v in sorted(k.items(), key=lambda kv:-kv[1]['ms'])[:6]])"; done
python bench.py --workload dof6-proof --steps 1 --warmup 0 > gpurun_out/r2_h_dof6-proof.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/r2_h_dof6-proof.json')); print('dof6-proof', d['value'], d['config']['verified'], d['config']['iterations'], d['device_share'])"
