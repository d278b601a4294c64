#!/bin/bash
# Occupancy / unroll sweep of the batched FISTA step kernel (bf_step): builds one
# library per (min CTAs per SM, elements per trip) from the objects of the last
# full build and times config 5 with each (run the loop part on the GPU box).
#   tools/bf_variants.sh build      # here
#   tools/bf_variants.sh run        # on the GPU box
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/scratch
VARS="1_4 3_4 3_2 4_4 4_2 4_1 5_2 5_1 6_2"
if [ "$1" = build ]; then
  for v in $VARS; do
    mb=${v%_*}; un=${v#*_}
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -Iinclude \
      --expt-relaxed-constexpr -DBF_MINB=$mb -DBF_UNROLL=$un -c paper_1007_3753_b200/csrc/batch_fista.cu -o /tmp/bf_$v.o
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/scratch/lib_bf_$v.so \
      $(ls build/*.o | grep -v batch_fista.o) /tmp/bf_$v.o
  done
else
  for v in $VARS; do
    echo "== min CTAs/SM ${v%_*}, elements per trip ${v#*_}"
    for cfg in "8192 float32" "1024 float32" "1024 float64"; do
      ELL1_LIB_PATH=$PWD/tools/scratch/lib_bf_$v.so python tools/fista32_breakdown.py $cfg 2>&1 | grep -E "^B=|bf_step"
    done
  done
fi
