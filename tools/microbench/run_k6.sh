timeout 900 ncu --set full --import-source on --clock-control none -k regex:kron_rot_kernel -c 1 -o /tmp/k6_fold python tools/microbench/rot_one.py 9d > /tmp/k6.log 2>&1
KRONOP_KRON_FOLD=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:kron_rot_kernel -c 1 -o /tmp/k6_dense python tools/microbench/rot_one.py 9d > /tmp/k6b.log 2>&1
for r in k6_fold k6_dense; do python tools/ncu_summary.py /tmp/$r.ncu-rep gpurun_out/$r.json > /dev/null; ncu -i /tmp/$r.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip -c > gpurun_out/${r}_src.csv.gz; ncu -i /tmp/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null; done
cat gpurun_out/k6_fold.json gpurun_out/k6_dense.json
