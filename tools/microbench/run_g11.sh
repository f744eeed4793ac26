python tools/microbench/rot_bench.py 2>&1 | tail -1
KRONOP_ROT_CT=0 python tools/microbench/rot_bench.py 2>&1 | tail -1
python -m pytest tests/test_gpu_switches.py tests/test_gpu_config_parity.py -k "switch or config5_group or full_size or qhop" -q 2>&1 | tail -3
