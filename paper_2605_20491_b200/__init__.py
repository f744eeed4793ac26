"""B200-native tensor-product Schrodinger solver (drop-in for the hot path of arxiv/paper_2605_20491).

The product is libkronop.so (sm_100a CUDA kernels + C++ host setup behind the C-ABI in
include/kronop_cuda.h); `api` is the Python mirror of the reference operator API used by tests and
bench.py.
"""
from ._lib import LIB_PATH, KronopError, ParameterError, NumericalError, CapabilityError, lib  # noqa
