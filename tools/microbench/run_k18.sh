# ncu captures of the Kronecker kernels (9D DFMA group, 6D DMMA group) and the bench launch list
timeout 900 ncu --set full --import-source on --clock-control none -k regex:kron_rot_kernel -c 1 -o /tmp/r02_kron9 python tools/microbench/rot_one.py 9d > /tmp/a.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:kron_dmma_kernel -c 1 -o /tmp/r02_kron6 python tools/microbench/rot_one.py 6d > /tmp/b.log 2>&1
for r in r02_kron9 r02_kron6; do python tools/ncu_summary.py /tmp/$r.ncu-rep gpurun_out/$r.json > /dev/null; done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file /tmp/r02b_ncu_launches.csv python bench.py --steps 2 --warmup 1 --no-extras --no-cpu > /tmp/ncu_bench.log 2>&1
cp /tmp/r02b_ncu_launches.csv gpurun_out/r02b_ncu_launches.csv
python tools/ncu_launch_summary.py gpurun_out/r02b_ncu_launches.csv gpurun_out/r02b_ncu_launches_summary.json ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv python bench.py --steps 2 --warmup 1 --no-extras --no-cpu > /dev/null
cat gpurun_out/r02_kron9.json gpurun_out/r02_kron6.json | grep -E "duration|dram|pipe|warps_active"
