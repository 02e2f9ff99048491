#!/bin/bash
# tests + bench + per-config table + ncu of the top kernel
PAT=${1:-star_pair}
make -C oracle -s
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
timeout 900 python tools/bench_all.py --steps 5 --no-cpu > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo rc=$? >> gpurun_out/configs.err
python tools/prof_stencil.py heat_3d 512 3 > gpurun_out/plain2.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:$PAT -c 2 -o gpurun_out/prof_top python tools/prof_stencil.py heat_3d 512 3 > gpurun_out/ncu2.log 2>&1
echo done
