#!/bin/bash
# Build shard.cu variants of the config-4 GEMV^T stream pipeline (columns per
# A stage CB, rows per chunk RC, column blocks per staged r chunk GB, A ring
# depth STA) as standalone libraries and time ell1_gemv / ell1_gemv_t at the
# 64 GiB single-GPU shape (diagnostics).
#   bash tools/gts_variants.sh > gpurun_out/gts.txt
set -e
cd "$(dirname "$0")/.."
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -fmad=false --expt-relaxed-constexpr -Iinclude -shared"
for v in "4 4096 4 2" "4 4096 6 2" "2 4096 8 3" "2 4096 6 3" "4 4096 5 2" "3 4096 6 2"; do
  set -- $v
  nvcc $F -DELL1_GTS_CB=$1 -DELL1_GTS_RC=$2 -DELL1_GTS_GB=$3 -DELL1_GTS_STA=$4 paper_1007_3753_b200/csrc/shard.cu -o /tmp/libgts_$1_$2_$3_$4.so
  echo "CB=$1 RC=$2 GB=$3 STA=$4"
  python tools/gemv_bench.py --full --lib /tmp/libgts_$1_$2_$3_$4.so
done
