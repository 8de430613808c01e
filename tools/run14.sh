for sl in 0 40 100 300 1000; do echo "sleep $sl"; for w in 15 63 101; do RMGPU_PHASE_SLEEP=$sl timeout 120 python tools/time_morph.py 4096 4096 $w $w 0 1; done; done
