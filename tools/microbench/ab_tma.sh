# A/B of TMA pass-kernel variants on one box: per-pass times of the 1024^3 solve
export CPLX=${CPLX:-0}
for L in ${LIBS:-tools/microbench/libs/tma_r01.so paper_2605_20491_b200/libkronop.so tools/microbench/libs/tma_r01.so paper_2605_20491_b200/libkronop.so}; do
  echo "== $L"
  KRONOP_LIB=$L python tools/microbench/solve_passes.py 2>&1 | tail -1
done
