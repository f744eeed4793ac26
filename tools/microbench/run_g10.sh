python tools/microbench/solve_passes.py 2>&1 | tail -1
KRONOP_ROTATE_PASSES=0 python tools/microbench/solve_passes.py 2>&1 | tail -1
python tools/microbench/solve_passes.py 2>&1 | tail -1
python -m pytest tests -m gpu -q -x 2>&1 | tail -4
