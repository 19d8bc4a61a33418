#!/bin/bash
# Experiments: tile width sweep + ncu of the Cholesky kernels.
mkdir -p gpurun_out
python -m paper_2203_11875_b200._build
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "condensed or full" 2>&1 | tail -3 > gpurun_out/pytest_exp.log
for c in 8 16 32; do
  PF_TILE_COLS=$c timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_c$c.json 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_chol_panel|k_chol_update|k_chol_solve" -s 20 -c 3 -f \
    -o gpurun_out/prof_chol python bench.py --profile-steps 1 --delta-w 1e6 > gpurun_out/ncu_chol.log 2>&1
cat gpurun_out/pytest_exp.log
