for l in "" tools/variants/kr_c1s4.so tools/variants/kr_t3c3s3.so tools/variants/kr_t3c2s4.so; do
  for f in 1 0; do KRONOP_KRON_FOLD=$f KRONOP_LIB=$l python tools/microbench/kron_bench.py 9d | sed "s/^/fold=$f /"; done
done
