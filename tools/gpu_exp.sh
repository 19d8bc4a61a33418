#!/bin/bash
# Experiments over prebuilt libraries build/libpf_<tag>.so (LIBS) x tile widths (CS).
mkdir -p gpurun_out
for tag in ${LIBS}; do for c in ${CS:-32 64}; do
  PF_LIB=build/libpf_$tag.so PF_TILE_COLS=$c timeout 200 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-generic ${EXP_ARGS} \
     > gpurun_out/exp_${tag}_c$c.json 2>&1
  python -c "import json,sys; d=json.load(open('gpurun_out/exp_${tag}_c$c.json')); k=d['roofline']['per_kernel']; print('$tag c=$c', round(d['value']), ' '.join('%s=%.2f'%(a,b['ms']) for a,b in k.items()))" || tail -3 gpurun_out/exp_${tag}_c$c.json
done; done
