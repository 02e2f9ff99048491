cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_r2.py tests/test_abi.py -q -x -k "halo or abi or declared or workspace" 2>&1 | tail -3
