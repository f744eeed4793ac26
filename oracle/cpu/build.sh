#!/bin/sh
# CPU oracle (C++ restatement of the reference CPU path) -> oracle/cpu/build/libkronop_cpu.so.
# Same flags as the reference's Release build (proj/CMakeLists.txt:9: -O3, no -march) + OpenMP.
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
mkdir -p "$HERE/build"
g++ -O3 -std=c++20 -fopenmp -fPIC -shared -Wall -o "$HERE/build/libkronop_cpu.so.tmp" \
    "$HERE/kronop_cpu.cpp" -ldl
mv "$HERE/build/libkronop_cpu.so.tmp" "$HERE/build/libkronop_cpu.so"
