#!/bin/bash
# A/B of sweep variants (build/libpf_<tag>.so): short bench timings + one ncu --set full of k_fwd and k_adj each.
mkdir -p gpurun_out
for tag in ${LIBS}; do
  PF_LIB=build/libpf_$tag.so timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-generic --no-next > gpurun_out/exp_$tag.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/exp_$tag.json')); k=d['roofline']['per_kernel']; print('$tag', round(d['value']), ' '.join('%s=%.2f'%(a,b['ms']) for a,b in k.items()))" || tail -3 gpurun_out/exp_$tag.json
done
if [ -n "$NCU" ]; then for tag in ${NCU}; do
  PF_LIB=build/libpf_$tag.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fwd|k_adj" -c 2 -f \
    -o gpurun_out/prof_sw_$tag python bench.py --profile-steps 1 --no-cpu-baseline --no-e2e --no-generic --no-next > gpurun_out/ncu_sw_$tag.log 2>&1
  tail -2 gpurun_out/ncu_sw_$tag.log
done; fi
