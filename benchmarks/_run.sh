set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/r2_gputest1.log; cat gpurun_out/r2_gputest1.log
for w in dof4-proof dof5-proof; do python bench.py --workload $w --steps 2 --warmup 1 > gpurun_out/r2_bench_$w.json 2> gpurun_out/r2_bench_$w.err; tail -c 900 gpurun_out/r2_bench_$w.json; tail -2 gpurun_out/r2_bench_$w.err; done
python bench.py --workload dof6-proof --steps 1 --warmup 0 > gpurun_out/r2_bench_dof6-proof.json 2> gpurun_out/r2_bench_dof6-proof.err; tail -c 1200 gpurun_out/r2_bench_dof6-proof.json; tail -2 gpurun_out/r2_bench_dof6-proof.err
PERMATRACE_B200_SOLVE_LOG=2 timeout 500 python benchmarks/proof_run.py --dof 6 --clutter 3 --lam 0.5 --gamma 0.35 --samples 1000 --feedback-cap 2000 --push-mult 2.15 --max-iters 40 --timeout 450 > gpurun_out/r2_sweep9_1.log 2>&1; grep -v "^Traceback\|^  " gpurun_out/r2_sweep9_1.log | tail -2 | cut -c1-600
