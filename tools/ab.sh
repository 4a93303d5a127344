cd $GRAFT_REPO_ROOT
for i in 1 2; do
for pr in 0 1; do echo "PAIR=$pr"; for b in 17 34 100; do EPS_GEMM_PAIR=$pr python tools/timeline.py $b 2>&1 | grep "step span"; done; done
done
