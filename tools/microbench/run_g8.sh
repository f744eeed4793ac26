timeout 900 ncu --set full --import-source on --clock-control none -k regex:fused_rot_kernel -c 1 -o gpurun_out/r02_rot9 python tools/microbench/rot_one.py 9d > gpurun_out/r02_rot9.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fused_rot_kernel -c 1 -o gpurun_out/r02_rot6 python tools/microbench/rot_one.py 6d > gpurun_out/r02_rot6.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:mode_product_tma -c 3 -o gpurun_out/r02_solve_passes env CPLX=0 N=1024 python tools/microbench/solve_passes.py > gpurun_out/r02_solve_ncu.log 2>&1
python tools/config4_histories.py 3 41 > gpurun_out/r02_config4_histories.json 2> gpurun_out/r02_config4_histories.err
tail -c 600 gpurun_out/r02_config4_histories.json
