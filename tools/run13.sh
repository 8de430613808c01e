timeout 800 python -m pytest tests -m gpu -q --timeout=300 -x -k "sweep or random_medium or golden or cfg" > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log; grep -E "FAILED|Error" gpurun_out/t.log | head -5
for w in 9 15 21 31 63 101; do timeout 120 python tools/time_morph.py 4096 4096 $w $w 0 1; done
timeout 120 python tools/time_morph.py 16384 16384 101 101 0 1
for rh in 128 192 320; do RMGPU_STREAM_RH=$rh timeout 120 python tools/time_morph.py 4096 4096 63 63 0 1; done
