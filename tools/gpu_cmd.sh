python -m pytest tests -m gpu -q -x > gpurun_out/r2_gpu_all.log 2>&1
