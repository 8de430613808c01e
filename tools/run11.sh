timeout 300 ncu --set full --import-source on --clock-control none -k regex:morph_phase -s 4 -c 1 -o gpurun_out/ph63n -f python tools/time_morph.py 4096 4096 63 63 0 1 --nograph > gpurun_out/ncu_a.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:morph_phase -s 4 -c 1 -o gpurun_out/ph15n -f python tools/time_morph.py 4096 4096 15 15 0 1 --nograph > gpurun_out/ncu_b.log 2>&1
tail -1 gpurun_out/ncu_a.log
