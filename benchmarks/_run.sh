set -x
cd /root/repo
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "taylor or full_size_refine or ill_conditioned or large_support" -s 2>&1 | grep -v "^$" | tail -30 > gpurun_out/r2_taylor_test2.log; cat gpurun_out/r2_taylor_test2.log
for w in dof6 dof6-s4096 dof6-s16384 dof5; do python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2_c_$w.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/r2_c_$w.json')); k=d['kernels']; print('$w', round(d['ms_per_step'],2), d['config'].get('rows_left_to_evaluation_kernels'), d['roofline']['frac'], [(n, round(v['ms'],2)) for n,v in sorted(k.items(), key=lambda kv:-kv[1]['ms'])[:6]])"; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'pt_ref_edges|pt_dedup_round|pt_dedup_follow|pt_ref_extract|pt_check32' -c 6 -o gpurun_out/r2_refine2_full python bench.py --steps 1 --warmup 0 --kernel-only > /dev/null 2>&1
ncu -i gpurun_out/r2_refine2_full.ncu-rep --page raw --csv > gpurun_out/r2_refine2_full_raw.csv
