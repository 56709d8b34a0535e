#!/bin/bash
# A/B the tuning variants in build/variants/ with the config-2 bench (twice each).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do
for lib in build/variants/lib_*.so; do
  name=$(basename $lib .so)
  STRAGGLAR_LIB=$PWD/$lib timeout 300 python bench.py --no-cpu --steps 10 --warmup 3 > gpurun_out/tune_$name.json 2> gpurun_out/tune_$name.err
  python -c "
import json,sys
d=json.load(open('gpurun_out/tune_$name.json'))
print('$name', 'B', d['value'], 'A', d['T_phaseA_us'], 'ring', d['ring_us'], 'direct', d['direct_completion']['T_post_us'], 'frac', d['roofline']['frac'], 'G', d['config']['slices_per_rank'])
" || echo "$name failed: $(tail -2 gpurun_out/tune_$name.err)"
done
done
