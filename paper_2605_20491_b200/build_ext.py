"""Build libkronop.so in-tree: nvcc for the sm_100a CUDA sources, g++ (C++20) for the host setup.

The shared library is the C-ABI boundary declared in include/kronop_cuda.h. It links the CUDA
runtime statically, so loading it (and calling the host-setup entry points) works on a machine
without a GPU. Usage: python -m paper_2605_20491_b200.build_ext [--force]
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libkronop.so")
BUILD = os.path.join(HERE, "_build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU = ["mode_product.cu", "mode_product_tma.cu", "fused_rot.cu", "vector_ops.cu", "capi.cu", "drivers.cu", "fieldio.cu", "tc_lowp.cu", "ozaki.cu", "slab.cu", "kron_prop.cu"]
CPP = ["host_setup.cpp"]


def _run(cmd):
    print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)


def build(force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = [os.path.join(CSRC, f) for f in CU + CPP]
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp"))]
    hdrs.append(os.path.join(HERE, "..", "include", "kronop_cuda.h"))
    newest = max(os.path.getmtime(p) for p in srcs + hdrs + [os.path.abspath(__file__)])
    if not force and os.path.exists(OUT) and os.path.getmtime(OUT) >= newest:
        return OUT
    jobs = []
    for f in CU:
        o = os.path.join(BUILD, f + ".o")
        jobs.append(([NVCC, *ARCH, "-O3", "-std=c++20", "-lineinfo", "-Xcompiler", "-fPIC",
                      "-Xcompiler", "-fopenmp", "--expt-relaxed-constexpr", "-c",
                      os.path.join(CSRC, f), "-o", o], o))
    for f in CPP:
        o = os.path.join(BUILD, f + ".o")
        jobs.append((["g++", "-O3", "-std=c++20", "-fPIC", "-fopenmp", "-Wall", "-c",
                      os.path.join(CSRC, f), "-o", o], o))
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=len(jobs)) as ex:
        list(ex.map(lambda j: _run(j[0]), jobs))
    objs = [o for _, o in jobs]
    tmp = OUT + ".tmp"
    _run([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-Xcompiler", "-fopenmp",
          "-cudart", "static"])
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv)
