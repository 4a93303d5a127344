cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -n 2
for i in 1 2; do
for pdl in 0 1; do echo "PDL=$pdl"; EPS_PDL=$pdl python tools/timeline.py 17 2>&1 | grep "step span"; EPS_PDL=$pdl python tools/timeline.py 400 2>&1 | grep "step span"; done
done
