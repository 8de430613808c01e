timeout 800 python -m pytest tests -m gpu -q --timeout=300 -x -k "small_window or golden or random_medium or band or batched or cfg1" > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log; grep -E "FAILED|Error" gpurun_out/t.log | head -5
for L in default B; do
  if [ $L = default ]; then unset RMGPU_LIB_PATH; else export RMGPU_LIB_PATH=$PWD/exp/lib$L.so; fi
  echo "== $L"
  for w in 3 5 7; do timeout 120 python tools/time_morph.py 4096 4096 $w $w 0 1; timeout 120 python tools/time_morph.py 16384 16384 $w $w 0 1; done
  timeout 120 python tools/time_morph.py 4096 4096 3 3 0 2
  timeout 120 python tools/time_morph.py 4096 4096 7 7 0 2
done
