#!/bin/bash
# Round-end measurement set: GPU tests, smoke, default bench line, configs 2-4, reference arm,
# ncu launch list and full captures of the reduction and Cholesky kernels.
mkdir -p gpurun_out
python -m paper_2203_11875_b200._build > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
for c in case118 case1354 case2869; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$c.json 2>> gpurun_out/bench.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --profile-steps 1 > gpurun_out/ncu_launch.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k_fwd|k_blk|k_adj|k_proj" -c 6 -f \
    -o gpurun_out/prof_reduce python bench.py --profile-steps 1 > gpurun_out/ncu_full.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k_chol_dag|k_lu\b|k_chol_unpack" -c 3 -f \
    -o gpurun_out/prof_chol python bench.py --profile-steps 1 > gpurun_out/ncu_chol.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log | tail -2; cat gpurun_out/bench.json | head -c 600; echo; tail -3 gpurun_out/bench.err
