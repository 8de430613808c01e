timeout 900 python -m pytest tests -m gpu -q --timeout=300 -x -k "small_window or golden or random_medium or band or batched or cfg1 or degenerate or padding" > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log; grep -E "FAILED|Error" gpurun_out/t.log | head -5
RMGPU_FORCE_KERNEL=1 timeout 120 python tools/time_morph.py 16384 16384 1 1 0 1
RMGPU_FORCE_KERNEL=1 timeout 120 python tools/time_morph.py 4096 4096 1 1 0 1
timeout 120 python tools/time_morph.py 16384 16384 1 3 0 1
timeout 120 python tools/time_morph.py 16384 16384 3 3 0 1
