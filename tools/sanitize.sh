#!/bin/bash
# compute-sanitizer sweep over the hand-written kernels at small shapes
# (VERDICT r01 item 8): memcheck, racecheck, synccheck, initcheck on the
# single-instance persistent kernels (software grid barrier, engine.cuh),
# the tcgen05 3xTF32 GEMM (mbarrier/TMEM ring, DSMEM split-K) and the
# batched solvers.  Logs go to gpurun_out/sanitize/<tool>_<group>.log.
set -u
OUT=${OUT:-gpurun_out/sanitize}
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
declare -A SEL
SEL[fista]="tests/test_fista_gpu.py -k small_1400 or qr or zero_rhs or budget_cap"
SEL[dalm]="tests/test_dalm_gpu.py -k small_1700 or zero_data or two_variable"
SEL[homotopy]="tests/test_homotopy_gpu.py -k small_1300 or identity or zero_rhs"
SEL[tc3]="tests/test_tc_gemm_gpu.py"
SEL[batched]="tests/test_batched_gpu.py"
SEL[sharded]="tests/test_sharded_gpu.py"
SEL[misc]="tests/test_numerics_gpu.py"
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  for g in ${GROUPS_:-fista dalm homotopy tc3 batched sharded misc}; do
    sel=${SEL[$g]}
    file=${sel%% *}
    k=""
    if [[ "$sel" == *" -k "* ]]; then k=${sel#* -k }; fi
    log="$OUT/${tool}_${g}.log"
    echo "== $tool $g" | tee "$log"
    if [ -n "$k" ]; then
      timeout ${TMO:-900} $CS --tool $tool --print-limit 50 --error-exitcode 99 \
        python -m pytest "$file" -k "$k" -x -q -p no:cacheprovider >> "$log" 2>&1
    else
      timeout ${TMO:-900} $CS --tool $tool --print-limit 50 --error-exitcode 99 \
        python -m pytest "$file" -x -q -p no:cacheprovider >> "$log" 2>&1
    fi
    rc=$?
    echo "rc=$rc" >> "$log"
    echo "$tool $g rc=$rc $(grep -m1 -E 'ERROR SUMMARY|passed|failed' "$log" | head -1)"
  done
done
