cd $GRAFT_REPO_ROOT
for e in "RMGPU_FUSE=0" "RMGPU_FUSE=1 RMGPU_SEP_HH=0" "RMGPU_FUSE=0 RMGPU_SEP_HH=0"; do
  echo -n "cfg4 $e : "; env $e timeout 300 python bench.py --workload cfg4 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e --no-self-check --soak-seconds 0 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step'],3))"
done
for W in 21; do for F in 0 1; do echo -n "u16 1024x1024 x512 erode fuse=$F: "; RMGPU_FUSE=$F python tools/time_morph.py 4096 4096 $W $W 0 2 | cut -c1-150; done; done
