cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -n 1
for i in 1 2; do
python tools/gemm_bench.py fwd_qkv fwd_fc1_gelu2 fwd_proj fwd_fc2
EPS_LIB_PATH=$PWD/tools/_cmp/libeps_b200_base.so python tools/gemm_bench.py fwd_qkv fwd_fc1_gelu2 fwd_proj fwd_fc2
done
