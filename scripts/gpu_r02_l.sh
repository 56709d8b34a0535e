#!/bin/bash
# Per-process sub-slice default at system scope: MPS-shared ranks, sub 1 vs 16,
# config 2 (256 MiB fp32) and 1 GiB bf16, n = 4 and 8, two repetitions.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02l}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; exit 1; }
for rep in 1 2; do
 for wl in config2 config3_1GiB; do
  for n in 4 8; do
   for sub in 1 16; do
    STRAGGLAR_SUBSLICES=$sub timeout 900 python bench.py --gpus $n --mps --steps 10 --warmup 3 --workload $wl --no-cpu > gpurun_out/${T}_${wl}_n${n}_sub${sub}_$rep.json 2> gpurun_out/${T}_${wl}_n${n}_sub${sub}_$rep.err
    echo "$wl n=$n sub=$sub rep=$rep rc=$? $(python -c "
import json;d=json.loads(open('gpurun_out/${T}_${wl}_n${n}_sub${sub}_$rep.json').read().strip().splitlines()[-1]);print(d['value'], d['T_phaseA_us'], {k:v['T_post_us'] for k,v in d['algorithms'].items()})" 2>&1 | tail -1)"
   done
  done
 done
done
