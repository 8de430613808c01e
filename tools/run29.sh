timeout 120 python tools/time_morph.py 1920 1080 3 3 0 1
RMGPU_COL_BLOCKS=2 timeout 120 python tools/time_morph.py 1920 1080 3 3 0 1
timeout 120 python tools/time_morph.py 1920 1080 3 3 1 1
timeout 900 python -m pytest tests -m gpu -q --timeout=300 -x -k "cfg1 or small_window or golden" 2>&1 | tail -2
