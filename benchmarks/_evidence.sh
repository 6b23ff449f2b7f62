set -x
cd /root/repo
python benchmarks/bfs_scaling.py --dim 6 --lambdas 0.14 0.1 --reps 2 > gpurun_out/r2_bfs_scaling.jsonl 2> gpurun_out/r2_bfs_scaling.err; cut -c1-700 gpurun_out/r2_bfs_scaling.jsonl
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'pt_wave_probe|pt_wave_partner|pt_wave_admit|pt_wave_count|pt_rehash' --launch-skip 50 -c 10 -o gpurun_out/r2_bfs_full python benchmarks/bfs_scaling.py --dim 6 --lambdas 0.14 --reps 1 > /dev/null 2>&1
ncu -i gpurun_out/r2_bfs_full.ncu-rep --page raw --csv > gpurun_out/r2_bfs_full_raw.csv
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'pt_cell_cofaces|pt_ref_edges|pt_ref_vertices|pt_ref_signs|pt_dedup_round|pt_dedup_follow|pt_ref_extract' -c 8 -o gpurun_out/r2_stress_full python bench.py --workload dof6-stress --steps 1 --warmup 0 --kernel-only > /dev/null 2>&1
ncu -i gpurun_out/r2_stress_full.ncu-rep --page raw --csv > gpurun_out/r2_stress_full_raw.csv
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 1 --warmup 1 --kernel-only > /dev/null 2>&1
for w in dof3 dof4 dof5 dof6-stress dof6-stress1g dof6-s4096 dof6-s16384; do python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_line_$w.json 2> gpurun_out/r2_line_$w.err; python -c "
import json,sys; d=json.load(open('gpurun_out/r2_line_$w.json')); print('$w', round(d['ms_per_step'],2), round(d['value']/1e9,3), 'e2e', round(d['e2e']['value']/1e9,3), d['clocks'].get('hbm_used_max_gb'), d['config']['crossing_fine_edges'], d['config']['points_checked'])"; done
python bench.py --workload dof3-proof --steps 2 --warmup 1 > gpurun_out/r2_bench_dof3-proof.json 2>/dev/null; tail -c 700 gpurun_out/r2_bench_dof3-proof.json
python bench.py > gpurun_out/r2_line_dof6.json 2> gpurun_out/r2_line_dof6.err; tail -c 600 gpurun_out/r2_line_dof6.json
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r2_line_dof6_reference.json 2>/dev/null; tail -c 400 gpurun_out/r2_line_dof6_reference.json
timeout 1500 compute-sanitizer --tool memcheck python bench.py --workload dof4 --steps 1 --warmup 0 --kernel-only > gpurun_out/r2_memcheck_dof4.log 2>&1; tail -4 gpurun_out/r2_memcheck_dof4.log
timeout 1500 compute-sanitizer --tool racecheck python bench.py --workload dof4 --steps 1 --warmup 0 --kernel-only > gpurun_out/r2_racecheck_dof4.log 2>&1; tail -4 gpurun_out/r2_racecheck_dof4.log
