#!/usr/bin/env bash
# Round measurement recipe (run on a B200 box through gpurun, from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 1800 -- 'bash tools/gpu_round.sh'
# Writes gpurun_out/b_<workload>.json (bench lines), gpurun_out/launches_cfg2.csv (ncu launch list of
# the default bench) and two ncu --set full captures of the dominant kernels. Summaries that are
# judged are copied into profiles/ by hand (tools/ncu_summary.py, tools/ncu_mix.py).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout=300 > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/b_cfg2.json 2> gpurun_out/b_cfg2.err
for w in cfg1 cfg3 cfg4 cfg5; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/b_$w.json 2> gpurun_out/b_$w.err
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/b_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv \
  --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  --soak-seconds 0 > gpurun_out/ncu_launch.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:morph_col -s 8 -c 1 \
  -o gpurun_out/col3 -f python tools/time_morph.py 4096 4096 3 3 0 1 --nograph > gpurun_out/ncu_col.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"pass_kernel|vtma" -s 4 -c 2 \
  -o gpurun_out/sep63 -f python tools/time_morph.py 4096 4096 63 63 0 1 --nograph > gpurun_out/ncu_sep.log 2>&1
