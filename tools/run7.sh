timeout 800 python -m pytest tests -m gpu -q --timeout=300 -x -k "small_window or golden or random_medium or band or batched or cfg1" > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log; grep -E "FAILED|Error" gpurun_out/t.log | head -5
for m in 2 3 4 6 8; do echo "blocks=$m"; for w in 3 7; do RMGPU_COL_BLOCKS=$m timeout 120 python tools/time_morph.py 4096 4096 $w $w 0 1; done; done
timeout 120 python tools/time_morph.py 16384 16384 3 3 0 1
timeout 120 python tools/time_morph.py 16384 16384 7 7 0 1
