#!/bin/bash
# Build an experimental libmwb variant into exp/ (git-ignored, travels to the GPU box):
#   scripts/build_variant.sh NAME [-DKNOB=VALUE ...]
# then run a script with MWB_LIB=$PWD/exp/libmwb_NAME.so (development aid).
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p exp
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  --expt-relaxed-constexpr --extended-lambda -Xcompiler -fPIC,-O2 -shared "$@" -I include \
  paper_1709_02549_b200/csrc/mwb_kernels.cu -o exp/libmwb_$name.so
echo exp/libmwb_$name.so
