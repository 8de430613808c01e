timeout 800 python -m pytest tests -m gpu -q --timeout=300 > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log; grep -E "FAILED" gpurun_out/t.log | head
timeout 300 ncu --set full --import-source on --clock-control none -k regex:morph_col -s 8 -c 1 -o gpurun_out/col3 -f python tools/time_morph.py 4096 4096 3 3 0 1 --nograph > gpurun_out/ncu_col3.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:morph_col -s 8 -c 1 -o gpurun_out/col7 -f python tools/time_morph.py 4096 4096 7 7 0 1 --nograph > gpurun_out/ncu_col7.log 2>&1
tail -2 gpurun_out/ncu_col3.log
