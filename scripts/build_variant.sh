#!/usr/bin/env bash
# Build an A/B variant of the library: bash scripts/build_variant.sh <name> [-DFLAG ...]
# -> build/<name>.so (time it with: bash scripts/ab.sh <config> build/<name>.so ...)
set -e
name=$1; shift
mkdir -p build
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -cudart static -shared \
  -Xcompiler -fPIC,-O3 "$@" -o build/$name.so paper_2512_09664_b200/csrc/pivgen_b200.cu
echo built build/$name.so
