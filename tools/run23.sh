timeout 120 python tools/copy_floor.py 4096 4096 1
timeout 120 python tools/copy_floor.py 1920 1080 1
timeout 120 python tools/copy_floor.py 16384 16384 1
timeout 120 python tools/copy_floor.py 1024 1024 2
RMGPU_FORCE_KERNEL=1 timeout 120 python tools/time_morph.py 4096 4096 1 1 0 1
RMGPU_FORCE_KERNEL=1 timeout 120 python tools/time_morph.py 16384 16384 1 1 0 1
for m in 1 2 3; do RMGPU_COL_BLOCKS=$m timeout 120 python tools/time_morph.py 4096 4096 3 3 0 1; done
