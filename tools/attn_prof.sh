cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/attn_bench.py vit-b16 bert-base-384 bert-large-128 > gpurun_out/attn_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_bwd_fused -s 3 -c 1 -o gpurun_out/prof_attn_bwd -f python tools/attn_bench.py vit-b16 > gpurun_out/ncu_attn_bwd.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_fwd_persistent -s 3 -c 1 -o gpurun_out/prof_attn_fwd -f python tools/attn_bench.py vit-b16 > gpurun_out/ncu_attn_fwd.log 2>&1
cat gpurun_out/attn_bench.log
