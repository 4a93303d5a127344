#!/bin/bash
# One gpurun session: tests, smoke, bench, ncu launch list + full captures.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
if [ "${NCU:-1}" = "1" ]; then
B="python bench.py --steps 1 --warmup 1 --no-schedule --no-cpu"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch_bench.log 2>&1
# one step of block GEMMs (layer 1 forward: QKV, proj, FC1, FC2) + attention + LayerNorm
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 5 -c 4 -o gpurun_out/prof_gemm -f $B > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 1 -c 1 -o gpurun_out/prof_attn -f $B > gpurun_out/ncu_attn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_bwd -s 1 -c 1 -o gpurun_out/prof_attnb -f $B > gpurun_out/ncu_attnb.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ln_fwd -s 4 -c 1 -o gpurun_out/prof_ln -f $B > gpurun_out/ncu_ln.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ln_bwd -s 4 -c 1 -o gpurun_out/prof_lnb -f $B > gpurun_out/ncu_lnb.log 2>&1
timeout 600 python tools/timeline.py 400 > gpurun_out/timeline.txt 2>&1
python tools/step_breakdown.py > gpurun_out/step_breakdown.txt 2>&1
fi
tail -n 3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench.err
cat gpurun_out/bench.json
