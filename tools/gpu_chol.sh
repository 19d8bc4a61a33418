#!/bin/bash
# Cholesky experiments: chol_bench timings (head vs current), a task trace, the GPU Cholesky tests.
mkdir -p gpurun_out
for b in ${CHOL_BINS:-chol_bench_head chol_bench}; do echo "== $b"; timeout 120 ./tools/$b.bin 2889 8 6 | tail -2; done
timeout 120 ./tools/chol_bench_trace.bin 2889 8 3 gpurun_out/chol_trace.csv | tail -1
python tools/chol_trace.py gpurun_out/chol_trace.csv > gpurun_out/chol_trace_summary.txt 2>&1; cat gpurun_out/chol_trace_summary.txt | head -30
timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 -k "${PYTEST_K:-condensed or full_size}" 2>&1 | tail -4
