for L in paper_2605_20491_b200/libkronop.so tools/microbench/libs/rot_nosplit3.so tools/microbench/libs/rot_split3_128.so paper_2605_20491_b200/libkronop.so; do KRONOP_LIB=$L python tools/microbench/rot_bench.py 2>&1 | tail -1; done
python -m pytest tests/test_gpu_config_parity.py -k "config5_group or full_size or qhop or criterion8" -q 2>&1 | tail -3
python -m pytest tests/test_gpu_parity.py -k "small_extent or high_dimensional" -q 2>&1 | tail -3
