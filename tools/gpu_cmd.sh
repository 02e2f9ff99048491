python -m pytest tests/test_gpu_r2.py tests/test_gpu.py -q -x -k "group or lockstep" > gpurun_out/r2_slab_tests.log 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --force-slab > gpurun_out/r2_bench_slab1.log 2>&1
