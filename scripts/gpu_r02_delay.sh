#!/bin/bash
# Partial-overlap regime on the per-process path (N2): 8 ranks under
# MPS, config 2, straggler delay D swept; completion from the non-stragglers'
# start (T_total) for every algorithm.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02r}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; exit 1; }
for d in 0 100 200 300 400 500 700 1000; do
  timeout 900 python bench.py --gpus 8 --mps --steps 10 --warmup 3 --no-cpu --delay-us $d > gpurun_out/${T}_mps8_d$d.json 2> gpurun_out/${T}_mps8_d$d.err
  echo "d=$d rc=$? $(python -c "
import json;d=json.loads(open('gpurun_out/${T}_mps8_d$d.json').read().strip().splitlines()[-1]);print(d['T_phaseA_nodelay_us'], {k:(v['T_total_us'], v['T_post_us']) for k,v in d['algorithms'].items()})" 2>&1 | tail -1)"
done
