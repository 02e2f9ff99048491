python -m pytest tests/test_gpu.py tests/test_gpu_r2.py -q -x -k "heat or jacobi or golden or stencil or medium" > gpurun_out/r2_chain_tests.log 2>&1
python tools/bench_all.py --no-cpu --steps 20 --only C2/heat_3d,C1/jacobi_2d > gpurun_out/r2_chain.jsonl 2> gpurun_out/r2_chain.err
GFB_STENCIL_CHAIN=0 python tools/bench_all.py --no-cpu --steps 20 --only C2/heat_3d >> gpurun_out/r2_chain.jsonl 2>> gpurun_out/r2_chain.err
