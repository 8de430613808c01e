cd $GRAFT_REPO_ROOT
t() { echo -n "$* : "; env "$@" python tools/time_morph.py $S $S $W $W 1 1 | cut -c1-160; }
for W in 15 31 63 101; do S=4096 t RMGPU_FUSE=1; done
S=4096 W=63 t RMGPU_FUSE_NT=2
S=4096 W=63 t RMGPU_FUSE_PF=1
S=32768 W=63 t RMGPU_FUSE=1
python tools/trace_fuse.py 4096 4096 63 63 1 50 > gpurun_out/tr63.txt 2>&1
timeout 300 python tools/fuse_check.py --quick 2>&1 | head -1
