cd $GRAFT_REPO_ROOT
t() { echo -n "$* : "; env "$@" timeout 60 python tools/time_morph.py $S $S $W $W 1 1 | cut -c1-160; }
for W in 15 31 63 101; do S=4096 t RMGPU_FUSE=1; done
S=4096 W=63 t RMGPU_FUSE_PAIR=1
S=32768 W=63 t RMGPU_FUSE=1
S=32768 W=63 t RMGPU_FUSE_PAIR=1
for d in 1 2 3; do S=32768 W=63 t RMGPU_FUSE_DBG=$d; done
timeout 300 python tools/fuse_check.py --quick 2>&1 | head -1
