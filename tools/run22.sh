timeout 900 python -m pytest tests -m gpu -q --timeout=300 -x -k "transpose or cfg3 or golden" > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log; grep -E "FAILED|Error|assert" gpurun_out/t.log | head -5
timeout 600 python bench.py --workload cfg3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_cfg3.json 2> gpurun_out/b_cfg3.err
python -c "
import json; d=json.loads(open('gpurun_out/b_cfg3.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac']); [print(w) for w in d['per_window']]"
