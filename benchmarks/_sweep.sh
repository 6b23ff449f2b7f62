cd /root/repo
export PERMATRACE_B200_SOLVE_LOG=2
i=0
run() { i=$((i+1)); timeout 400 python benchmarks/proof_run.py "$@" --max-iters 40 --timeout 360 > gpurun_out/r2_sweep10_$i.log 2>&1; echo "== $i: $@"; grep -v "^Traceback\|^  " gpurun_out/r2_sweep10_$i.log | tail -2 | cut -c1-500; }
run --dof 6 --clutter 2 --lam 0.5 --gamma 0.35 --samples 1000 --feedback-cap 2000 --push-mult 2.15
run --dof 6 --clutter 3 --lam 0.5 --gamma 0.35 --samples 1000 --feedback-cap 2000 --push-mult 2.15 --rng-seed 1
run --dof 6 --clutter 3 --lam 0.5 --gamma 0.5 --samples 1000 --feedback-cap 2000 --push-mult 1.8
run --dof 6 --clutter 3 --lam 0.5 --gamma 0.35 --samples 1000 --feedback-cap 2000 --push-mult 2.15 --scene-seed 5
run --dof 6 --clutter 4 --lam 0.5 --gamma 0.35 --samples 1000 --feedback-cap 2000 --push-mult 2.15 --scene-seed 3
