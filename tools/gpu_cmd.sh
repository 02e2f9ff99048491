cd $GRAFT_REPO_ROOT/tools/lab
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"sgemm_tma" --launch-skip 2 -c 1 -o ../../gpurun_out/mm4_k64 python mm_one.py 4096 4096 64 1 0 > ../../gpurun_out/ncu_mm4.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"sgemm_tma" --launch-skip 2 -c 1 -o ../../gpurun_out/mm4_w2 python mm_one.py 64 4096 4096 0 0 > ../../gpurun_out/ncu_mm4b.log 2>&1
ls ../../gpurun_out | grep mm4
