#!/bin/bash
# K5 granularity sweep at 4096^2 (no rebuild: planner knobs only)
t() { python tools/time_morph.py "$@" 2>&1 | tail -1 | awk '{print $6, $7}'; }
for w in 63 15; do
echo "== 4096^2 ${w}x${w}: K3"; RMGPU_CHAIN=0 t 4096 4096 $w $w 1 1
for parts in 2 5 10; do for rb in 40 80; do for lag in 2 4 8 40; do
  echo -n "parts=$parts rb=$rb lag=$lag: "
  RMGPU_CHAIN=1 RMGPU_SEP_PARTS=$parts RMGPU_CHAIN_RB=$rb RMGPU_CHAIN_SMIN=$rb RMGPU_CHAIN_LAG=$lag t 4096 4096 $w $w 1 1
done; done; done
done
