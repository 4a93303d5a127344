cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -n 2
A_ENV=EPS_GEMM_PAIR=0 ROWS=1 bash tools/ab_timeline.sh
timeout 600 python bench.py --no-schedule --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['kernels']['gemm'])"
