#!/bin/bash
# Builds a variant of the library for same-box A/B runs: tools/build_variant.sh OUT.so [nvcc flags]
cd "$(dirname "$0")/.."
out=$1; shift
exec /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC,-O3 -Xptxas -v --expt-relaxed-constexpr -shared "$@" -ccbin g++ -o "$out" \
  paper_1502_02941_b200/csrc/*.cu paper_1502_02941_b200/csrc/*.cpp
