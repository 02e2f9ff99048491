#!/bin/bash
# One gpurun call: tests, bench line, per-config table, launch list and a
# full ncu capture of the top kernel. Outputs land in gpurun_out/ (scratch);
# tools/summarize_profiles.py turns them into profiles/ summaries.
cd "$(dirname "$0")/.."
make -C oracle -s
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err; echo rc=$? >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.jsonl 2> gpurun_out/bench_ref.err
# the slab-decomposition path at one rank (communication-free rewrite, graph captured)
timeout 600 python bench.py --force-slab --steps 5 --no-cpu-baseline > gpurun_out/bench_slab1.jsonl 2> gpurun_out/bench_slab1.err
timeout 1500 python tools/bench_all.py --steps 10 --plans > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
timeout 600 python tools/op_table.py > gpurun_out/ops.txt 2>&1
# launch list of the bench command (cold-cache serialised times: compare shares)
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
# full capture of the fused stencil kernel: steady launches (skip the first
# forward timestep, whose boundary copies are not yet in place)
python tools/prof_stencil.py heat_3d 512 4 > gpurun_out/plain2.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:star_pair --launch-skip 1 -c 4 \
  -o gpurun_out/prof_top python tools/prof_stencil.py heat_3d 512 4 > gpurun_out/ncu2.log 2>&1
# the mlp GEMMs: the W2 forward (skinny, weight-streaming) and W2 gradient (K = 64)
(cd tools/lab && python mm_time.py > ../../gpurun_out/mm_time.log 2>&1)
for sh in "64 4096 4096 0 0" "4096 4096 64 1 0"; do
  tag=$(echo $sh | tr ' ' _)
  (cd tools/lab && timeout 300 ncu --set full --clock-control none -k regex:sgemm_tma --launch-skip 2 -c 1 \
    -o ../../gpurun_out/gemm_$tag python mm_one.py $sh > ../../gpurun_out/ncu_gemm_$tag.log 2>&1)
done
echo done
