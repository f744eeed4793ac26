for r in 1 2; do for l in "" tools/variants/mp_head.so; do KRONOP_LIB=$l python tools/microbench/solve_passes.py 2>/dev/null | head -c 600; echo " [$l]"; done; done
timeout 900 ncu --set full --clock-control none -k regex:mode_product_tma -c 1 -o /tmp/r02_rot_solve_u python tools/microbench/solve_once.py > /tmp/a.log 2>&1
python tools/ncu_summary.py /tmp/r02_rot_solve_u.ncu-rep gpurun_out/r02_rotated_pass_units.json > /dev/null; grep -E "duration|dram|dmma_pipe" gpurun_out/r02_rotated_pass_units.json
python -m pytest tests/test_gpu_parity.py -q -x -k "mode_product or separable or c1 or host" 2>&1 | tail -1
