#!/bin/bash
# usage: tools/sweep_rh.sh W H wx wy elem "rh list"
for rh in $6; do
  RMGPU_STREAM_RH=$rh python tools/time_morph.py $1 $2 $3 $4 0 $5
done
