#!/bin/bash
# ncu --set full of the reduction kernels (one launch each) on the default bench workload.
mkdir -p gpurun_out
python -m paper_2203_11875_b200._build > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-k_blk}" -c ${NCU_C:-1} -f \
    -o gpurun_out/prof_${NCU_TAG:-hvp} python bench.py --profile-steps 1 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
