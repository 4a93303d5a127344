cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_pipeline_gpu.py tests/test_trainer_gpu.py tests/test_vit_gpu.py -x -q 2>&1 | tail -n 3
timeout 900 python tools/measured_report.py r01e 3 > gpurun_out/mr.log 2>&1; grep -v Warn gpurun_out/mr.log | tail -n 3
