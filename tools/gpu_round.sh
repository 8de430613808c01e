#!/usr/bin/env bash
# Round measurement recipe (run on a B200 box through gpurun, from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 3000 -- "bash tools/gpu_round.sh"
# GPU tests, the bench line of every workload and of the reference arm, the ncu launch list of the
# default bench, one ncu --set full capture of the separable passes, per-op DRAM traffic, the pipe
# issue-rate microbenchmark, copy floors and the PCIe probe -> gpurun_out/ (summaries that are judged
# are copied into profiles/ by hand).
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout=600 > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/b_cfg2.json 2> gpurun_out/b_cfg2.err; tail -c 200 gpurun_out/b_cfg2.err
for w in cfg1 cfg3 cfg4 cfg5; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/b_$w.json 2> gpurun_out/b_$w.err; tail -c 200 gpurun_out/b_$w.err
done
timeout 400 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/b_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv \
  --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  --no-self-check --soak-seconds 0 > gpurun_out/ncu_launch.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"pass_kernel" -s 4 -c 2 \
  -o gpurun_out/sep63 -f python tools/time_morph.py 4096 4096 63 63 0 1 --nograph > gpurun_out/ncu_sep.log 2>&1
python tools/ops_once.py cfg2 > gpurun_out/ops_cfg2.txt 2>&1 && \
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none \
  --clock-control none --csv --log-file gpurun_out/traffic_cfg2.csv python tools/ops_once.py cfg2 > gpurun_out/ncu_traffic.log 2>&1
tools/ubench/pipes > gpurun_out/ubench_pipes.txt 2>&1
for s in "4096 4096 1" "1920 1080 1" "8192 8192 1" "4096 4096 2"; do timeout 60 python tools/copy_floor.py $s; done > gpurun_out/copy_floor.txt 2>&1
timeout 100 python tools/pcie_probe2.py > gpurun_out/pcie_probe.txt 2>&1
ls gpurun_out
