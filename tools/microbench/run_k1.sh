# Kronecker propagate: parity tests, then timing A/B (T-form vs Kronecker), then Strang steps/s
python -m pytest tests/test_gpu_kron.py -x -q 2>&1 | tail -15
python -m pytest tests/test_gpu_switches.py -x -q -k "KRON or SPEC_SPLIT" 2>&1 | tail -3
python -m pytest tests/test_gpu_parity.py -x -q -k "small_extent or high_dim or degenerate or qhop or evolve" 2>&1 | tail -3
KRONOP_KRON_PROP=0 python tools/microbench/rot_bench.py > gpurun_out/k1_rot_tform.json 2>&1
python tools/microbench/rot_bench.py > gpurun_out/k1_rot_kron.json 2>&1
cat gpurun_out/k1_rot_tform.json gpurun_out/k1_rot_kron.json
for f in 0 1; do KRONOP_BPHASE_FUSED=$f python tools/microbench/bphase_bench.py; done > gpurun_out/k1_bphase.json 2>&1
cat gpurun_out/k1_bphase.json
