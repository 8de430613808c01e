#!/bin/bash
# per-op timings of the cfg2 windows (+ u16 21x21, big images with --big): tools/quick_times.sh [--big]
t() { timeout 120 python tools/time_morph.py "$@" 2>&1 | tail -1 | awk '{print $1, $2, $6, $7, $10, $11}'; }
for w in 15 31 63 101; do t 4096 4096 $w $w 1 1; done
t 4096 4096 1 31 1 1; t 4096 4096 31 1 1 1; t 4096 4096 3 3 1 1; t 4096 4096 7 7 1 1
t 4096 4096 21 21 0 2
if [ "$1" = "--big" ]; then t 16384 16384 63 63 1 1; t 32768 32768 63 63 1 1; fi
