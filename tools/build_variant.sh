#!/bin/bash
# Build a variant of libsphbi_cuda.so with extra nvcc flags (code-shape
# experiments): tools/build_variant.sh <name> [-DFOO=1 ...] -> _variants/<name>.so
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p _variants
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -lineinfo -std=c++17 --shared \
  -Xcompiler -fPIC -Xptxas -v "$@" paper_2507_21686_b200/csrc/sphbi_cuda.cu -o _variants/$name.so \
  > _variants/$name.log 2>&1
echo "_variants/$name.so"
