cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu.py -q -x -k "3xtf32 or mlp or C4" > gpurun_out/t_mm.log 2>&1; tail -3 gpurun_out/t_mm.log
cd tools/lab && python mm_time.py 2>&1 | tee ../../gpurun_out/mm_time_mn.log
