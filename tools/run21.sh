timeout 600 python bench.py --workload cfg4 --steps 5 --warmup 3 > gpurun_out/b_cfg4.json 2> gpurun_out/b_cfg4.err
timeout 600 python bench.py --workload cfg3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b_cfg3.json 2> gpurun_out/b_cfg3.err
