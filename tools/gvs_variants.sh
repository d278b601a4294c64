#!/bin/bash
# Variants of the config-4 streamed GEMV partial pass (columns per stage CB,
# rows per chunk RC, ring depth ST) timed at the 64 GiB shape (diagnostics).
set -e
cd "$(dirname "$0")/.."
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -fmad=false --expt-relaxed-constexpr -Iinclude -shared -lcuda"
for v in "4 4096 3" "2 8192 3" "8 2048 3" "4 4096 2" "2 4096 6" "1 16384 3"; do
  set -- $v
  nvcc $F -DELL1_GVS_CB=$1 -DELL1_GVS_RC=$2 -DELL1_GVS_ST=$3 paper_1007_3753_b200/csrc/shard.cu -o /tmp/libgvs_$1_$2_$3.so
  echo "CB=$1 RC=$2 ST=$3"
  python tools/gemv_bench.py --full --lib /tmp/libgvs_$1_$2_$3.so
done
