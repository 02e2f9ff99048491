#!/bin/bash
# star-pair iteration: parity vs oracle, GPU tests, bench, ncu of the top kernel
make -C oracle -s
timeout 300 python tools/check_star.py > gpurun_out/check_star.log 2>&1; echo rc=$? >> gpurun_out/check_star.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
python tools/prof_stencil.py heat_3d 512 3 > gpurun_out/plain2.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:star_pair -c 4 -o gpurun_out/prof_top python tools/prof_stencil.py heat_3d 512 3 > gpurun_out/ncu2.log 2>&1
echo done
