python -m pytest tests/test_gpu_r2.py tests/test_gpu.py -q -x -k "heat or c5 or jacobi or stencil or slab or lockstep" > gpurun_out/r2_star_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/r2_star_tests.log 2>&1
for lib in build/variants/libgfb_ns.so paper_2509_02197_b200/libgfb.so; do
GFB_LIBRARY=$lib python tools/time_star.py >> gpurun_out/r2_time.log 2>&1
done
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
timeout 300 ncu --metrics $M --clock-control none -k regex:star_pair -c 6 --csv python tools/prof_stencil.py heat_3d 512 4 > gpurun_out/r2_ncu_st.csv 2>&1
