#!/bin/bash
# GEMM A/B of two library builds on the same box: interleaved rounds of
# tools/gemm_bench.py for the named shapes (default: the GELU / gelu' epilogues).
# usage: tools/gemm_ab.sh A.so B.so [shapes...]
cd "$(dirname "$0")/.."
A=$1; B=$2; shift 2
SH=${@:-b400_fwd_fc1 b400_dgrad_fc2}
for r in 1 2 3; do
  for L in $A $B; do
    echo "== $L"
    EPS_LIB_PATH=$(readlink -f $L) python tools/gemm_bench.py $SH
  done
done
