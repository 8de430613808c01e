timeout 900 python -m pytest tests -m gpu -q -x --timeout=300 2>&1 | tail -5
for w in 3 5 7 15 63 101; do timeout 120 python tools/time_morph.py 4096 4096 $w $w 0 1; done
timeout 120 python tools/time_morph.py 4096 4096 3 3 0 1 --nograph
timeout 120 python tools/time_morph.py 1920 1080 3 3 0 1
timeout 120 python tools/time_morph.py 16384 16384 3 3 0 1
timeout 120 python tools/time_morph.py 16384 16384 7 7 0 1
timeout 120 python tools/time_morph.py 4096 4096 3 3 0 2
timeout 120 python tools/time_morph.py 4096 4096 7 7 0 2
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_r01b.json 2> gpurun_out/bench_r01b.err
python -c "
import json; d=json.load(open('gpurun_out/bench_r01b.json')); print(d['value'], d['roofline']['frac'], d['ms_per_step'], d['gpu_launches']); [print(w) for w in d['per_window']]"
