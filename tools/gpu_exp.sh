#!/bin/bash
# Experiments: dot width (compile-time) x tile width (run-time) for the sweeps.
mkdir -p gpurun_out
python -m paper_2203_11875_b200._build
SRC=paper_2203_11875_b200/csrc
for dw in 2 4 8; do
  nvcc -shared -Xcompiler -fPIC -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -DPF_DOT_W=$dw \
    -o /tmp/libpf_dw$dw.so $SRC/pf_plan.cpp $SRC/pf_eval.cu $SRC/pf_reduce.cu $SRC/pf_chol.cu $SRC/pf_api.cu
done
for dw in 2 4 8; do for c in 32 64; do
  PF_LIB=/tmp/libpf_dw$dw.so PF_TILE_COLS=$c timeout 200 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e \
     > gpurun_out/exp_dw${dw}_c$c.json 2>&1
done; done
