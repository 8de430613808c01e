timeout 300 ncu --set full --import-source on --clock-control none -k regex:morph_col -s 2 -c 1 -o gpurun_out/col3_16k -f python tools/time_morph.py 16384 16384 3 3 0 1 --nograph > gpurun_out/ncu_a.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:morph_col -s 8 -c 1 -o gpurun_out/col3c -f python tools/time_morph.py 4096 4096 3 3 0 1 --nograph > gpurun_out/ncu_b.log 2>&1
tail -1 gpurun_out/ncu_a.log
