timeout 800 python -m pytest tests -m gpu -q --timeout=300 -x > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log; grep -E "FAILED|Error" gpurun_out/t.log | head
for w in 3 5 7; do timeout 120 python tools/time_morph.py 4096 4096 $w $w 0 1; done
timeout 120 python tools/time_morph.py 1920 1080 3 3 0 1
timeout 120 python tools/time_morph.py 16384 16384 3 3 0 1
timeout 120 python tools/time_morph.py 16384 16384 7 7 0 1
timeout 120 python tools/time_morph.py 4096 4096 3 3 0 2
timeout 120 python tools/time_morph.py 4096 4096 7 7 0 2
timeout 300 ncu --set full --import-source on --clock-control none -k regex:morph_col -s 8 -c 1 -o gpurun_out/col3b -f python tools/time_morph.py 4096 4096 3 3 0 1 --nograph > gpurun_out/ncu_col3.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:morph_col -s 8 -c 1 -o gpurun_out/col7b -f python tools/time_morph.py 4096 4096 7 7 0 1 --nograph > gpurun_out/ncu_col7.log 2>&1
