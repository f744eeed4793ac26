for v in 2 0 1; do KRONOP_ROT_SPEC_SPLIT=$v python tools/microbench/rot_bench.py 2>&1 | tail -1; done
