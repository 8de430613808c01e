cd $GRAFT_REPO_ROOT
for a in "4096 4096 63 63" "4096 4096 15 15" "2048 2048 63 63" "1024 1024 63 63" "4096 512 63 63" "512 4096 63 63" "4096 4096 31 31"; do
  echo -n "$a : "; timeout 60 python tools/one_morph.py $a 0 1 2>&1 | tail -1 | cut -c1-150
done
for a in "4096 4096 63 63" ; do
  echo -n "nt2 $a : "; RMGPU_FUSE_NT=2 timeout 60 python tools/one_morph.py $a 0 1 2>&1 | tail -1 | cut -c1-150
  echo -n "nt4 $a : "; RMGPU_FUSE_NT=4 timeout 60 python tools/one_morph.py $a 0 1 2>&1 | tail -1 | cut -c1-150
  echo -n "pf1 $a : "; RMGPU_FUSE_PF=1 timeout 60 python tools/one_morph.py $a 0 1 2>&1 | tail -1 | cut -c1-150
  echo -n "pf2 $a : "; RMGPU_FUSE_PF=2 timeout 60 python tools/one_morph.py $a 0 1 2>&1 | tail -1 | cut -c1-150
done
