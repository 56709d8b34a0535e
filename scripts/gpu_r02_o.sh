#!/bin/bash
# Sub-slice target size by message size (team mode): config 4 (25 MiB bf16),
# config 2 (256 MiB fp32), 1 GiB bf16.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02o}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; exit 1; }
run() {
  local name=$1 wl=$2; shift 2
  env "$@" timeout 600 python bench.py --no-cpu --steps 20 --warmup 5 --workload $wl > gpurun_out/${T}_$name.json 2> gpurun_out/${T}_$name.err
  echo "$name rc=$? $(python -c "import json;d=json.load(open('gpurun_out/${T}_$name.json'));print(d['value'], d['T_post_stats_us']['median'], d['T_phaseA_us'], d['fused_call']['us'], d['ring_us'], d['direct_completion']['T_post_us'])" 2>&1 | tail -1)"
}
for rep in 1 2; do
  for sb in 16384 32768 65536 131072; do run c4_sb${sb}_$rep config4 STRAGGLAR_SUBSLICE_BYTES=$sb; done
  for sb in 65536 131072 262144; do run c3_sb${sb}_$rep config3_1GiB STRAGGLAR_SUBSLICE_BYTES=$sb; done
done
