python -m pytest tests/test_gpu_r2.py -q -x -k "batch" > gpurun_out/r2_batch_tests.log 2>&1
