# ncu evidence for profiles/ (run on a GPU box from the repo root; each command ran clean first).
# Part A: bash tools/ncu_evidence.sh A  (traffic per cfg2 op, cfg2 launch list, cfg3 kernels)
# Part B: bash tools/ncu_evidence.sh B  (cfg4 and cfg5 kernels, one launch each)
set -u
mkdir -p gpurun_out
if [ "${1:-A}" = A ]; then
python tools/ops_once.py cfg2 > gpurun_out/ops_cfg2.txt 2>&1 && \
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none \
  --clock-control none --csv --log-file gpurun_out/traffic_cfg2.csv python tools/ops_once.py cfg2 > gpurun_out/ncu_traffic.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-self-check --soak-seconds 0 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_cfg2.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-self-check --soak-seconds 0 > gpurun_out/ncu_launch.log 2>&1
python tools/ops_once.py cfg3 > gpurun_out/ops_cfg3.txt 2>&1 && \
timeout 600 ncu --set full --clock-control none -k regex:"transpose_image|tiles" -c 4 \
  -o gpurun_out/cfg3 -f python tools/ops_once.py cfg3 --warm 0 > gpurun_out/ncu_cfg3.log 2>&1
else
python tools/ops_once.py cfg4 > gpurun_out/ops_cfg4.txt 2>&1 && \
timeout 600 ncu --set full --clock-control none -k regex:"pass_kernel" -s 1 -c 1 \
  -o gpurun_out/cfg4 -f python tools/ops_once.py cfg4 --warm 0 > gpurun_out/ncu_cfg4.log 2>&1
python tools/ops_once.py cfg5 > gpurun_out/ops_cfg5.txt 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:"vtma" -c 1 \
  -o gpurun_out/cfg5 -f python tools/ops_once.py cfg5 --warm 0 > gpurun_out/ncu_cfg5.log 2>&1
fi
ls -la gpurun_out
