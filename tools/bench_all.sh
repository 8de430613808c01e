# all bench workloads on one GPU (run from the repo root on a GPU box); lines to gpurun_out/b_*.json
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/b_cfg2.json 2> gpurun_out/b_cfg2.err; tail -c 300 gpurun_out/b_cfg2.err
for w in cfg1 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/b_$w.json 2> gpurun_out/b_$w.err; tail -c 300 gpurun_out/b_$w.err
done
timeout 600 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/b_ref.json 2>&1
