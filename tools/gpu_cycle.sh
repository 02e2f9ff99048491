#!/bin/bash
# One measurement cycle on the GPU box: parity tests, bench, launch list,
# ncu full capture of the top kernel (pattern $1, default star_pair).
PAT=${1:-star_pair}
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu1.log 2>&1
python tools/prof_stencil.py heat_3d 512 3 > gpurun_out/plain2.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:$PAT -c 2 -o gpurun_out/prof_top python tools/prof_stencil.py heat_3d 512 3 > gpurun_out/ncu2.log 2>&1
echo done
