"""Build a variant of libkronop.so in which one CUDA source is replaced (A/B experiments on the
GPU box in one run: KRONOP_LIB=<variant .so>). Usage:
  python tools/build_variant.py <replacement.cu> <which.cu> <out.so> [-DFLAG ...]
The other objects come from the in-tree build (paper_2605_20491_b200/_build)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_20491_b200 import build_ext as B  # noqa: E402

src, which, out = sys.argv[1:4]
flags = sys.argv[4:]
B.build()
obj = out + ".o"
subprocess.check_call([B.NVCC, *B.ARCH, "-O3", "-std=c++20", "-lineinfo", "-Xcompiler", "-fPIC",
                       "-Xcompiler", "-fopenmp", "--expt-relaxed-constexpr", "-I", B.CSRC, *flags,
                       "-c", src, "-o", obj])
objs = [obj if f == which else os.path.join(B.BUILD, f + ".o") for f in B.CU]
objs += [os.path.join(B.BUILD, f + ".o") for f in B.CPP]
subprocess.check_call([B.NVCC, *B.ARCH, "-shared", "-o", out, *objs, "-Xcompiler", "-fopenmp",
                       "-cudart", "static"])
os.remove(obj)
print(out)
