python -m pytest tests -m gpu -q -x > gpurun_out/r2_gpu_all.log 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench1.log 2>&1
