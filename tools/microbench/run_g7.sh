for L in paper_2605_20491_b200/libkronop.so tools/microbench/libs/rot_a.so tools/microbench/libs/rot_b.so tools/microbench/libs/rot_e.so paper_2605_20491_b200/libkronop.so; do KRONOP_LIB=$L python tools/microbench/rot_bench.py 2>&1 | tail -1; done
python tools/microbench/bphase_bench.py 2>&1 | tail -1
KRONOP_BPHASE_FUSED=0 python tools/microbench/bphase_bench.py 2>&1 | tail -1
python -m pytest tests/test_gpu_switches.py tests/test_gpu_config_parity.py::test_soft_coulomb_4d_99_matches_paper -v 2>&1 | tail -15
