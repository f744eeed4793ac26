"""Build tests/cpp/test_api.cpp against include/kronop/kronop.hpp + libkronop.so (CPU: compile
and link only) and run it on the GPU box."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_api.cpp")
LIBDIR = os.path.join(ROOT, "paper_2605_20491_b200")
EXE = os.path.join(ROOT, "tests", "cpp", "test_api")


def build():
    subprocess.check_call(["g++", "-std=c++20", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
                           SRC, "-o", EXE, "-L", LIBDIR, "-lkronop",
                           "-Wl,-rpath," + LIBDIR])
    return EXE


def test_cpp_api_compiles_and_links():
    assert os.path.exists(build())


@pytest.mark.gpu
def test_cpp_api_runs_reference_style_checks():
    exe = build()
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "all" in out.stdout and "checks passed" in out.stdout
