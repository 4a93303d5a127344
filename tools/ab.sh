cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -n 2
python tools/gemm_bench.py dgrad_fc2_mul fwd_fc1_gelu2 dgrad_proj_rowdot fwd_proj fwd_fc1_store dgrad_qkv wgrad_fc2
ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 3 -c 1 -o gpurun_out/prof_mul -f python tools/gemm_bench.py dgrad_fc2_mul > /dev/null 2>&1
