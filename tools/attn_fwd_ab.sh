#!/bin/bash
# Forward-kernel A/B: attention tests under each EPS_ATTN_FWD mode, then timing.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/attn_fwd_ab.log
: > $out
for m in ${MODES:-1 2}; do
  echo "== tests EPS_ATTN_FWD=$m" >> $out
  EPS_ATTN_FWD=$m timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k attention 2>&1 | tail -n 8 >> $out
done
for r in 1 2; do
  for m in 0 ${MODES:-1 2}; do
    echo "== bench EPS_ATTN_FWD=$m" >> $out
    EPS_ATTN_FWD=$m timeout 300 python tools/attn_bench.py vit-b16 bert-large-128 >> $out 2>&1
  done
done
cat $out
