python tools/microbench/rot_bench.py 2>&1 | tail -1
KRONOP_ROT_TMA_STORE=0 python tools/microbench/rot_bench.py 2>&1 | tail -1
python tools/microbench/rot_bench.py 2>&1 | tail -1
python -m pytest tests/test_gpu_config_parity.py -k "config5_group or full_size or qhop" -q 2>&1 | tail -2
python -m pytest tests/test_gpu_parity.py -k "small_extent or high_dimensional or folded or evolve or qhop" -q 2>&1 | tail -2
python -m pytest tests/test_gpu_switches.py tests/test_gpu_kernels.py -q 2>&1 | tail -2
