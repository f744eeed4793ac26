set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:kron_rot_kernel -c 1 -o /tmp/k2_kron9 python tools/microbench/rot_one.py 9d > /tmp/k2_kron9.log 2>&1
python tools/ncu_summary.py /tmp/k2_kron9.ncu-rep gpurun_out/k2_kron9.json > /dev/null
ncu -i /tmp/k2_kron9.ncu-rep --page source --csv --print-source sass > /tmp/k2_kron9_src.csv 2>/dev/null; gzip -c /tmp/k2_kron9_src.csv > gpurun_out/k2_kron9_src.csv.gz
ncu -i /tmp/k2_kron9.ncu-rep --page raw --csv > gpurun_out/k2_kron9_raw.csv 2>/dev/null
cat gpurun_out/k2_kron9.json
