cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_gemm_gpu.py tests/test_vit_gpu.py tests/test_bert_gpu.py -x -q 2>&1 | tail -n 4
python tools/attn_bench.py vit-b16 bert-large-128
python tools/attn_trace.py 2>/dev/null
timeout 600 python bench.py --no-schedule --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['kernels'])"
