#!/usr/bin/env bash
# Regenerates the round-2 evidence kept under profiles/ on a one-B200 box (run from the repo root, outputs in gpurun_out/):
#   gpurun --timeout 5400 -- 'bash benchmarks/evidence.sh'
# then copy / summarise with profiles/summarize.py as profiles/README.md describes.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
# dominant kernel + launch list of one step
# (the .ncu-rep files are exported to CSV and deleted: gpurun brings back at most 64 MiB)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pt_bisect_taylor -c 4 -o gpurun_out/taylor_full python bench.py --steps 1 --warmup 0 --kernel-only > /dev/null 2>&1
ncu -i gpurun_out/taylor_full.ncu-rep --page raw --csv > gpurun_out/taylor_full_raw.csv
ncu -i gpurun_out/taylor_full.ncu-rep --page source --csv --print-source cuda,sass --launch-skip 2 --launch-count 1 > gpurun_out/taylor_full_source.csv
rm -f gpurun_out/taylor_full.ncu-rep
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --kernel-only > /dev/null 2>&1
# hash / frontier kernels: BFS-only scaling, wave kernels of a mid-run wave, refine kernels at stress and bench size
python benchmarks/bfs_scaling.py --dim 6 --lambdas 0.14 0.1 --reps 2 > gpurun_out/bfs_scaling.jsonl
timeout 900 ncu --set full --clock-control none -k regex:'pt_wave_probe|pt_wave_partner|pt_wave_admit|pt_wave_count|pt_rehash' --launch-skip 50 -c 10 -o gpurun_out/bfs_full python benchmarks/bfs_scaling.py --dim 6 --lambdas 0.14 --reps 1 > /dev/null 2>&1
ncu -i gpurun_out/bfs_full.ncu-rep --page raw --csv > gpurun_out/bfs_full_raw.csv
rm -f gpurun_out/bfs_full.ncu-rep
timeout 1200 ncu --set full --clock-control none -k regex:'pt_cell_cofaces|pt_ref_vertices|pt_ref_signs' -c 6 -o gpurun_out/stress_full python bench.py --workload dof6-stress --steps 1 --warmup 0 --kernel-only > /dev/null 2>&1
ncu -i gpurun_out/stress_full.ncu-rep --page raw --csv > gpurun_out/stress_full_raw.csv
rm -f gpurun_out/stress_full.ncu-rep
timeout 900 ncu --set full --clock-control none -k regex:'pt_ref_edges|pt_dedup_round|pt_dedup_follow|pt_ref_extract|pt_check32' -c 6 -o gpurun_out/refine_full python bench.py --steps 1 --warmup 0 --kernel-only > /dev/null 2>&1
ncu -i gpurun_out/refine_full.ncu-rep --page raw --csv > gpurun_out/refine_full_raw.csv
rm -f gpurun_out/refine_full.ncu-rep
# bench lines: every workload, both arms of the headline one, the proofs, two ranks on one device
for w in dof3 dof4 dof5 dof6-stress dof6-stress1g dof6-s4096 dof6-s16384; do python bench.py --workload $w --steps 3 --warmup 3 > gpurun_out/line_$w.json 2> gpurun_out/line_$w.err; done
python bench.py > gpurun_out/line_dof6.json 2> gpurun_out/line_dof6.err
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/line_dof6_reference.json 2>/dev/null
for w in dof3-proof dof4-proof dof5-proof; do python bench.py --workload $w --steps 2 --warmup 1 > gpurun_out/proof_$w.json 2>/dev/null; done
python bench.py --workload dof6-proof --steps 1 --warmup 0 > gpurun_out/proof_dof6-proof.json 2>/dev/null
PT_BENCH_BACKEND=gloo python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/line_dof6_2ranks_1gpu.json 2>/dev/null
# sanitizers
timeout 1500 compute-sanitizer --tool memcheck python bench.py --workload dof4 --steps 1 --warmup 0 --kernel-only > gpurun_out/memcheck_dof4.log 2>&1
timeout 1500 compute-sanitizer --tool racecheck python bench.py --workload dof4 --steps 1 --warmup 0 --kernel-only > gpurun_out/racecheck_dof4.log 2>&1
timeout 1200 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -q -x -k "taylor and 3-700" > gpurun_out/memcheck_taylor.log 2>&1
tail -n 5 gpurun_out/memcheck_dof4.log gpurun_out/racecheck_dof4.log gpurun_out/memcheck_taylor.log
du -sh gpurun_out
