python -m pytest tests/test_gpu_kron.py -x -q 2>&1 | tail -2
python tools/microbench/kron_bench.py 9d
for f in 0 1; do KRONOP_BPHASE_FUSED=$f python tools/microbench/bphase_bench.py 2>/dev/null; done
