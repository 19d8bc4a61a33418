#!/bin/bash
# Quick GPU round-trip: build, selected GPU tests (PYTEST_K), short bench.
mkdir -p gpurun_out
python -m paper_2203_11875_b200._build > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout ${TEST_TIMEOUT:-300} python -m pytest tests -m gpu -q -x --timeout 200 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1
tail -15 gpurun_out/pytest_gpu.log
if [ -z "$NO_BENCH" ]; then
  timeout 300 python bench.py --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
  cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
fi
