cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_r2.py tests/test_gpu.py -q -k "finite_difference or batch" 2>&1 | grep -E "Error|assert|passed|failed" | head -30
