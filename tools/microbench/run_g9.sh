set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fused_rot_kernel -c 1 -o /tmp/r02_rot9 python tools/microbench/rot_one.py 9d > /tmp/r02_rot9.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fused_rot_kernel -c 1 -o /tmp/r02_rot6 python tools/microbench/rot_one.py 6d > /tmp/r02_rot6.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:mode_product_tma --launch-skip 4 -c 1 -o /tmp/r02_pass_a1 env CPLX=0 N=1024 python tools/microbench/solve_passes.py > /tmp/r02_pass_a1.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:mode_product_tma --launch-skip 8 -c 1 -o /tmp/r02_pass_div env CPLX=0 N=1024 python tools/microbench/solve_passes.py > /tmp/r02_pass_div.log 2>&1
for r in r02_rot9 r02_rot6 r02_pass_a1 r02_pass_div; do python tools/ncu_summary.py /tmp/$r.ncu-rep gpurun_out/$r.json > /dev/null; done
ncu -i /tmp/r02_rot9.ncu-rep --page source --csv --print-source sass > /tmp/r02_rot9_src.csv 2>/dev/null; gzip -c /tmp/r02_rot9_src.csv > gpurun_out/r02_rot9_src.csv.gz
ncu -i /tmp/r02_rot6.ncu-rep --page source --csv --print-source sass > /tmp/r02_rot6_src.csv 2>/dev/null; gzip -c /tmp/r02_rot6_src.csv > gpurun_out/r02_rot6_src.csv.gz
ls -la gpurun_out
python tools/microbench/cublas_passes.py > gpurun_out/r02_cublas_passes.json 2>&1
cat gpurun_out/r02_cublas_passes.json
python tools/config4_histories.py 3 41 > gpurun_out/r02_config4_histories.json 2> gpurun_out/r02_config4_histories.err
tail -c 300 gpurun_out/r02_config4_histories.json
