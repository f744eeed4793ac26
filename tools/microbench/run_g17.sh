for L in paper_2605_20491_b200/libkronop.so tools/microbench/libs/rot_noc2.so paper_2605_20491_b200/libkronop.so; do KRONOP_LIB=$L python tools/microbench/rot_bench.py 2>&1 | tail -1; done
python -m pytest tests/test_gpu_config_parity.py -k "config5_group or full_size or qhop" -q 2>&1 | tail -2
python -m pytest tests/test_gpu_parity.py -k "small_extent or high_dimensional or folded or evolve or qhop" -q 2>&1 | tail -2
