#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the small cases: smoke()
# (case9: every hot-path kernel incl. the LU cluster, the Cholesky DAG and the solves) and the
# case118 parity + NEXT-row tests (memcheck).
mkdir -p gpurun_out
python -m paper_2203_11875_b200._build > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
SMOKE='import __graft_entry__ as g; g.smoke()'
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -c "$SMOKE" > gpurun_out/san_${tool}_smoke.log 2>&1
  echo "$tool smoke rc=$?: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|smoke ok' gpurun_out/san_${tool}_smoke.log | tr '\n' ' ')"
done
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests -m gpu -q -x \
  -k "case118 or case9 or ipm or step" > gpurun_out/san_memcheck_tests.log 2>&1
echo "memcheck tests rc=$?: $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/san_memcheck_tests.log | tail -3 | tr '\n' ' ')"
