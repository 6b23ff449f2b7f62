cd /root/repo
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 | cut -c1-300
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
python bench.py --workload dof6-proof --steps 1 --warmup 0 > gpurun_out/r2_j_dof6-proof.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/r2_j_dof6-proof.json')); print('dof6-proof', d['value'], d['config']['verified'], d['config']['iterations'], d['device_share'], d['clocks'].get('hbm_used_max_gb'))"
