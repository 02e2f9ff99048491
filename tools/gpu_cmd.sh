cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_r2.py tests/test_gpu.py -q -x 2>&1 | tail -5
