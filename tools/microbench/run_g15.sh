python tools/configs_bench.py 3 5 3oz > gpurun_out/r02_configs.json 2> gpurun_out/r02_configs.err; tail -c 1500 gpurun_out/r02_configs.json
python tools/config5_bench.py both > gpurun_out/r02_config5_b.json 2> gpurun_out/r02_config5_b.err; tail -c 300 gpurun_out/r02_config5_b.json
