cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_r2.py -q -x -k "finite_difference" 2>&1 | tail -2
