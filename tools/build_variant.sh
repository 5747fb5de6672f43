#!/bin/bash
# Build a debug/experiment variant of the library into abtest/libhprime_<tag>.so
#   tools/build_variant.sh NOLDS -DHP_DBG_NOLDS
set -e
REPO=$(cd "$(dirname "$0")/.." && pwd)
tag=$1; shift
mkdir -p "$REPO/abtest"
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -shared -Xcompiler -fPIC \
  -cudart static "$@" -o "$REPO/abtest/libhprime_$tag.so" "$REPO/paper_2003_09133_b200/csrc/lfbp_capi.cu"
