python -m pytest tests/test_gpu_r2.py -q -x -k "config_scale" > gpurun_out/r2_plan_tests.log 2>&1
