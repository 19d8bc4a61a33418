#!/bin/bash
# GPU round-trip for measurement: default bench line, configs 2-4, reference arm (short), ncu launch list.
mkdir -p gpurun_out
python -m paper_2203_11875_b200._build > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 600 python bench.py --steps ${STEPS:-20} --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
for c in case118 case1354 case2869; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$c.json 2>> gpurun_out/bench.err
done
if [ -n "$REF" ]; then timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err; fi
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --profile-steps 1 > gpurun_out/ncu_launch.log 2>&1
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
