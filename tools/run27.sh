for w in 15 31 63 101; do timeout 120 python tools/time_morph.py 4096 4096 $w $w 0 1; done
timeout 120 python tools/time_morph.py 16384 16384 63 63 0 1
timeout 600 python -m pytest tests -m gpu -q --timeout=300 -x -k "sweep or random_medium" 2>&1 | tail -2
