# Round-end measurement set: the driver's bench command (both arms), and the ncu launch list of
# the bench's timed kernels (a number printed under ncu is never a bench value).
python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_n1.json 2> gpurun_out/r02_bench_n1.err
tail -c 400 gpurun_out/r02_bench_n1.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_bench_ref.json 2> gpurun_out/r02_bench_ref.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file /tmp/r02_ncu_launches.csv python bench.py --steps 2 --warmup 1 --no-extras --no-cpu > /tmp/ncu_bench.log 2>&1
cp /tmp/r02_ncu_launches.csv gpurun_out/r02_ncu_launches.csv
python tools/ncu_launch_summary.py gpurun_out/r02_ncu_launches.csv gpurun_out/r02_ncu_launches_summary.json ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv python bench.py --steps 2 --warmup 1 --no-extras --no-cpu > /dev/null
cat gpurun_out/r02_bench_n1.json | head -c 2500
cat gpurun_out/r02_bench_ref.json
