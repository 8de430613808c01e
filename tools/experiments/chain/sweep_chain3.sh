#!/bin/bash
t() { timeout 120 python tools/time_morph.py "$@" 2>&1 | tail -1 | awk '{print $6, $7}'; }
echo "== 32768^2 63"; RMGPU_CHAIN=0 t 32768 32768 63 63 1 1; RMGPU_CHAIN=1 t 32768 32768 63 63 1 1
for ah in 4 8 16 32; do echo -n "ahead=$ah "; RMGPU_CHAIN=1 RMGPU_CHAIN_AHEAD=$ah t 32768 32768 63 63 1 1; done
for roles in 84 64; do echo -n "roles=$roles "; RMGPU_CHAIN=1 RMGPU_CHAIN_ROLES=$roles t 32768 32768 63 63 1 1; done
echo -n "rbmax=160 "; RMGPU_CHAIN=1 RMGPU_CHAIN_RBMAX=160 t 32768 32768 63 63 1 1
echo -n "rbmax=320 "; RMGPU_CHAIN=1 RMGPU_CHAIN_RBMAX=320 t 32768 32768 63 63 1 1
echo "== 16384^2 63"; RMGPU_CHAIN=0 t 16384 16384 63 63 1 1; RMGPU_CHAIN=1 t 16384 16384 63 63 1 1
timeout 300 python tools/chain_check.py --time-only --cfg4 2>&1 | grep cfg4 | head -2
