cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_r2.py -q -x -k "concurrent_edges or lockstep or slab or group or c5 or heat" 2>&1 | tail -2
timeout 120 python tools/time_star.py
timeout 300 python tools/host_overhead.py 2>&1 | grep -E "single|slab rank 0 of"
