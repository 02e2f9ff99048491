cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu.py -q -x -k "3xtf32 or mlp or C4" 2>&1 | tail -2
cd tools/lab; for r in 1 2; do python mm_time.py 2>&1 | cut -c1-60; done
