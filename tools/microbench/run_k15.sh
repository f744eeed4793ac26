timeout 900 ncu --set full --import-source on --clock-control none -k regex:kron_dmma_kernel -c 1 -o /tmp/k15_d6 python tools/microbench/rot_one.py 6d > /tmp/k15.log 2>&1
python tools/ncu_summary.py /tmp/k15_d6.ncu-rep gpurun_out/k15_d6.json > /dev/null; ncu -i /tmp/k15_d6.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip -c > gpurun_out/k15_d6_src.csv.gz; ncu -i /tmp/k15_d6.ncu-rep --page raw --csv > gpurun_out/k15_d6_raw.csv 2>/dev/null
cat gpurun_out/k15_d6.json
