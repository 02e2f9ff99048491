python -m pytest tests/test_gpu_r2.py -q -x -k "measured_device" > gpurun_out/r2_mem_tests.log 2>&1
