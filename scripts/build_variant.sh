#!/usr/bin/env bash
# build_variant.sh NAME "-DFOO=1 -DBAR=2": in-tree libpbg variant for A/B runs (PBG_LIB=NAME)
set -e
cd "$(dirname "$0")/.."
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -I include -I paper_2002_11302_b200/csrc $2 -o paper_2002_11302_b200/$1 paper_2002_11302_b200/csrc/pbg.cu -lcudart
