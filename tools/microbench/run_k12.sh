python -m pytest tests/test_gpu_kron.py -x -q 2>&1 | tail -4
python tools/microbench/kron_bench.py 9d 6d
KRONOP_KRON_PROP=0 python tools/microbench/kron_bench.py 6d
