cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -q -x -k "transpose or cfg3" 2>&1 | tail -2
for b in 1 0; do RMGPU_TRANSPOSE_BFLY=$b python bench.py --workload cfg3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --soak-seconds 0 | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bfly=$b', round(d['value'],1), d['self_check']['bit_exact'], [(p['op'], p['us'], p['frac']) for p in d['per_window']])"; done
