timeout 900 python -m pytest tests -m gpu -q --timeout=300 -x > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log; grep -E "FAILED|Error" gpurun_out/t.log | head -5
for w in 9 15 31 63 101; do timeout 120 python tools/time_morph.py 4096 4096 $w $w 0 1; done
timeout 120 python tools/time_morph.py 4096 4096 1 31 0 1
timeout 120 python tools/time_morph.py 4096 4096 31 1 0 1
timeout 120 python tools/time_morph.py 16384 16384 63 63 0 1
