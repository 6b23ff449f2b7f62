export PERMATRACE_B200_SOLVE_LOG=2
i=0
run() { i=$((i+1)); timeout 330 python benchmarks/proof_run.py "$@" --max-iters 30 --timeout 300 > gpurun_out/r2_sweep8_$i.log 2>&1; echo "== $i: $@"; grep -v "^Traceback\|^  " gpurun_out/r2_sweep8_$i.log | tail -2 | cut -c1-600; }
run --dof 6 --clutter 0 --lam 0.5 --gamma 0.35 --samples 1500 --feedback-cap 2000 --push-mult 2.15 --limit 0.9
run --dof 6 --clutter 4 --lam 0.5 --gamma 0.35 --samples 1500 --feedback-cap 2000 --push-mult 2.15 --limit 0.9
run --dof 6 --clutter 0 --lam 0.5 --gamma 0.35 --samples 1000 --feedback-cap 2000 --push-mult 2.15
run --dof 4 --clutter 3 --lam 0.25 --gamma 0.5 --samples 2000 --feedback-cap 3000 --push-mult 2.5
run --dof 4 --clutter 3 --lam 0.3 --gamma 0.5 --samples 1500 --feedback-cap 2000 --push-mult 2.3
