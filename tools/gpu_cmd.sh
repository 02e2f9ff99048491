cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_r2.py -q -x -k "concurrent_edges or lockstep or slab or group" 2>&1 | tail -3
timeout 300 python tools/host_overhead.py 2>&1 | tail -12
