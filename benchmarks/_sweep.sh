export PERMATRACE_B200_SOLVE_LOG=2
i=0
run() { i=$((i+1)); timeout 330 python benchmarks/proof_run.py "$@" --max-iters 20 --timeout 300 > gpurun_out/r2_sweep7_$i.log 2>&1; echo "== $i: $@"; grep -v "^Traceback\|^  " gpurun_out/r2_sweep7_$i.log | tail -3 | cut -c1-600; }
run --dof 6 --clutter 0 --lam 0.5 --gamma 0.35 --samples 2000 --feedback-cap 2000 --push-mult 2.15
run --dof 6 --clutter 0 --lam 0.5 --gamma 0.35 --samples 2000 --feedback-cap 2000 --push-mult 1.9
run --dof 6 --clutter 0 --lam 0.6 --gamma 0.35 --samples 2000 --feedback-cap 2000 --push-mult 1.79
run --dof 5 --clutter 3 --lam 0.35 --gamma 0.5 --samples 2000 --feedback-cap 2000 --push-mult 2.5
run --dof 4 --clutter 3 --lam 0.25 --gamma 1.0 --samples 2000 --feedback-cap 3000 --push-mult 2.0
