timeout 600 python -m pytest tests -m gpu -q -x --timeout=300 -k "small_window_fuzz or golden or known or random_medium or degenerate or padding or cfg1 or batched or band" 2>&1 | tail -15
for w in 3 5 7; do timeout 120 python tools/time_morph.py 4096 4096 $w $w 0 1; done
timeout 120 python tools/time_morph.py 4096 4096 3 3 1 1
timeout 120 python tools/time_morph.py 16384 16384 3 3 0 1
timeout 120 python tools/time_morph.py 1920 1080 3 3 0 1
timeout 120 python tools/time_morph.py 4096 4096 3 3 0 2
timeout 120 python tools/time_morph.py 4096 4096 7 7 0 2
