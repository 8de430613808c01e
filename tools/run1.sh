set -x
timeout 900 python -m pytest tests -m gpu -q -x --timeout=300 2>&1 | tail -15
for w in 3 5 7 9 15 21 31 63 101; do timeout 120 python tools/time_morph.py 4096 4096 $w $w 0 1; done
timeout 120 python tools/time_morph.py 4096 4096 31 1 0 1
timeout 120 python tools/time_morph.py 4096 4096 1 31 0 1
timeout 120 python tools/time_morph.py 8192 8192 63 63 0 1
timeout 120 python tools/time_morph.py 16384 16384 3 3 0 1
timeout 120 python tools/time_morph.py 1024 1024 21 21 0 2
