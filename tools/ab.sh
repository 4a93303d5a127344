cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_kernels_gpu.py tests/test_vit_gpu.py -x -q 2>&1 | tail -n 2
for b in 17 50 400; do python tools/launch_overhead.py $b 2>&1 | grep batch; EPS_LIB_PATH=$PWD/tools/_cmp/libeps_b200_base.so python tools/launch_overhead.py $b 2>&1 | grep batch; done
