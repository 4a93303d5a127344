#!/bin/bash
# Attention-only GPU iteration: kernel tests, timing, optional ncu capture.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k attention > gpurun_out/attn_tests.log 2>&1; echo "rc=$?" >> gpurun_out/attn_tests.log
tail -n 15 gpurun_out/attn_tests.log
timeout 300 python tools/attn_bench.py vit-b16 bert-base-384 bert-large-128 2>&1 | tee gpurun_out/attn_bench.log
if [ "${NCU:-0}" = "1" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-attn_bwd_fused} -s 3 -c 1 -o gpurun_out/prof_attn_k -f python tools/attn_bench.py vit-b16 > gpurun_out/ncu_attn_k.log 2>&1
fi
