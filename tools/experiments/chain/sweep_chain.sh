#!/bin/bash
# K5 knob sweep on a GPU box: tools/sweep_chain.sh > gpurun_out/sweep_chain.log
t() { python tools/time_morph.py "$@" 2>&1 | tail -1; }
echo "== 32768^2 63x63 dilate"
RMGPU_CHAIN=0 t 32768 32768 63 63 1 1
echo -n "auto: "; RMGPU_CHAIN=1 t 32768 32768 63 63 1 1
for lag in 2 4 8 16; do
  for ctas in 4 3; do
    echo -n "lag=$lag ctas=$ctas: "; RMGPU_CHAIN=1 RMGPU_CHAIN_LAG=$lag RMGPU_CHAIN_CTAS=$ctas t 32768 32768 63 63 1 1
  done
done
for rb in 160 320; do
  echo -n "rbmax=$rb: "; RMGPU_CHAIN=1 RMGPU_CHAIN_RBMAX=$rb t 32768 32768 63 63 1 1
done
echo "== 16384^2 63x63 dilate"
RMGPU_CHAIN=0 t 16384 16384 63 63 1 1
RMGPU_CHAIN=1 t 16384 16384 63 63 1 1
echo "== 8192^2 63x63 dilate"
RMGPU_CHAIN=0 t 8192 8192 63 63 1 1
RMGPU_CHAIN=1 t 8192 8192 63 63 1 1
echo "== 4096^2"
for w in 15 63 101; do
  RMGPU_CHAIN=0 t 4096 4096 $w $w 1 1
  RMGPU_CHAIN=1 t 4096 4096 $w $w 1 1
  echo -n "lag=2: "; RMGPU_CHAIN=1 RMGPU_CHAIN_LAG=2 t 4096 4096 $w $w 1 1
done
python tools/chain_check.py --time-only --cfg4 2>&1 | grep cfg4
