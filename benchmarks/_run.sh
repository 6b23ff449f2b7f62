cd /root/repo
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 | cut -c1-300
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pt_bisect_taylor -c 4 -o gpurun_out/r2_taylor_v3 python bench.py --steps 1 --warmup 0 --kernel-only > /dev/null 2>&1; ncu -i gpurun_out/r2_taylor_v3.ncu-rep --page raw --csv > gpurun_out/r2_taylor_v3_raw.csv
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2_launches_v3.csv python bench.py --steps 1 --warmup 1 --kernel-only > /dev/null 2>&1
for w in dof3 dof4 dof5 dof6-stress dof6-stress1g dof6-s4096 dof6-s16384; do python bench.py --workload $w --steps 3 --warmup 3 > gpurun_out/r2_line_$w.json 2> gpurun_out/r2_line_$w.err; python -c "
import json,sys; d=json.load(open('gpurun_out/r2_line_$w.json')); print('$w', round(d['ms_per_step'],2), round(d['value']/1e9,3), 'e2e', round(d['e2e']['value']/1e9,3), d['clocks'].get('hbm_used_max_gb'), d['config']['crossing_fine_edges'], d['config']['points_checked'], d['config']['rows_left_to_evaluation_kernels'], d['parity_sample']['verdict'] if d.get('parity_sample') else None)"; done
python bench.py > gpurun_out/r2_line_dof6.json 2> gpurun_out/r2_line_dof6.err; python -c "
import json; d=json.load(open('gpurun_out/r2_line_dof6.json')); print('dof6', d['ms_per_step'], d['value'], d['e2e'], d['parity_sample']['verdict'], d['roofline']['frac'], d['roofline']['issue_frac'], d['cpu_baseline']['value'], d['cpu_baseline']['kind'])"
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r2_line_dof6_reference.json 2>/dev/null; tail -c 200 gpurun_out/r2_line_dof6_reference.json
for w in dof3-proof dof4-proof dof5-proof; do python bench.py --workload $w --steps 2 --warmup 1 > gpurun_out/r2_bench_$w.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/r2_bench_$w.json')); print('$w', d['value'], d['config']['verified'], d['config']['iterations'], d['config']['repeatable'], d['device_share'])"; done
python bench.py --workload dof6-proof --steps 1 --warmup 0 > gpurun_out/r2_bench_dof6-proof.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/r2_bench_dof6-proof.json')); print('dof6-proof', d['value'], d['config']['verified'], d['config']['iterations'], d['device_share'], d['clocks'].get('hbm_used_max_gb'))"
PT_BENCH_BACKEND=gloo python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2_line_dof6_2ranks_1gpu.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/r2_line_dof6_2ranks_1gpu.json')); print('2 ranks on one GPU', d['ms_per_step'], d['value'], d['config']['points_checked'])"
