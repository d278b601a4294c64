#!/bin/bash
# Build the whole library with extra nvcc defines into a scratch directory and
# run a command against it (diagnostics for engine tuning knobs, e.g.
# ELL1_GT_QU32):  bash tools/engine_variant.sh "-DELL1_GT_QU32=2" python bench.py --only-leg stream
set -e
cd "$(dirname "$0")/.."
DEFS="$1"; shift
OUT=/tmp/ell1_variant_$$
mkdir -p $OUT/pkg
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr $DEFS"
pids=()
for f in paper_1007_3753_b200/csrc/*.cu; do
  nvcc $F -c $f -o $OUT/$(basename $f .cu).o & pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libell1b200.so $OUT/*.o
cp -r paper_1007_3753_b200/*.py $OUT/pkg/ 2>/dev/null || true
ELL1_LIB_PATH=$OUT/libell1b200.so "$@"
