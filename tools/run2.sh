for w in 3 9 15 63 101; do timeout 120 python tools/time_morph.py 4096 4096 $w $w 0 1; done
timeout 120 python tools/time_morph.py 8192 8192 63 63 0 1
timeout 600 python bench.py > gpurun_out/bench_r01a.json 2> gpurun_out/bench_r01a.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1
