for m in 4 7 8 11 15 16; do RMGPU_COL_BLOCKS=$m RMGPU_FORCE_KERNEL=1 timeout 120 python tools/time_morph.py 16384 16384 1 1 0 1; done
for m in 7 16; do RMGPU_COL_BLOCKS=$m timeout 120 python tools/time_morph.py 16384 16384 3 3 0 1; done
