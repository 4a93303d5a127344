cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -k attention 2>&1 | tail -n 2
python tools/attn_bench.py vit-b16 bert-large-128
EPS_LIB_PATH=$PWD/tools/_cmp/libeps_b200_base.so python tools/attn_bench.py vit-b16 bert-large-128
python tools/attn_bench.py vit-b16 bert-large-128
