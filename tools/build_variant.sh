#!/bin/bash
# build/libpf_<tag>.so with extra nvcc flags: tools/build_variant.sh <tag> -DFOO=1 ...
tag=$1; shift
mkdir -p build
S=paper_2203_11875_b200/csrc
nvcc -shared -Xcompiler -fPIC -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a "$@" \
  -o build/libpf_$tag.so $S/pf_plan.cpp $S/pf_eval.cu $S/pf_reduce.cu $S/pf_chol.cu $S/pf_api.cu
