#!/bin/bash
# One GPU round-trip: parity tests (incl. full-size sampled), bench, ncu launch list + full captures.
mkdir -p gpurun_out
python -m paper_2203_11875_b200._build > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests -m gpu -q -x --timeout 200 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 400 python bench.py --steps ${STEPS:-10} --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --profile-steps 1 ${BENCH_ARGS} > gpurun_out/ncu_launch.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-k_fwd|k_blk|k_adj|k_proj}" -c ${NCU_C:-5} -f \
    -o gpurun_out/prof_reduce python bench.py --profile-steps 1 ${BENCH_ARGS} > gpurun_out/ncu_full.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k_chol_dag|k_lu\b|k_chol_pack|k_chol_unpack" -c 4 -f \
    -o gpurun_out/prof_chol python bench.py --profile-steps 1 ${BENCH_ARGS} > gpurun_out/ncu_chol.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
