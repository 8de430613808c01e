#!/usr/bin/env bash
# registers / spills of one K4 variant: tools/ptxas_check.sh SZ MAX B
R=/root/repo
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v \
  --expt-relaxed-constexpr -I $R/include -DFUSE_SZ=${1:-1} -DFUSE_MAX=${2:-0} -DFUSE_B=${3:-20} \
  -c $R/paper_2002_09474_b200/csrc/morph_fuse_inst.cu -o /tmp/fi.o 2>&1 | grep -E "error|Used|spill" | sort | uniq -c
