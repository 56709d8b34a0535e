#!/bin/bash
# Sub-slice target with the signalling warp (fences no longer on the copy-issuing thread).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02an}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; exit 1; }
run() {
  local name=$1 wl=$2; shift 2
  env "$@" timeout 600 python bench.py --no-cpu --steps 20 --warmup 5 --workload $wl > gpurun_out/${T}_$name.json 2> gpurun_out/${T}_$name.err
  echo "$name rc=$? $(python -c "import json;d=json.load(open('gpurun_out/${T}_$name.json'));print(d['value'], d['T_post_stats_us']['median'], d['fused_call']['us'])" 2>&1 | tail -1)"
}
for rep in 1 2; do
  for sb in 131072 65536 98304; do
    run c2_sb${sb}_$rep config2 STRAGGLAR_SUBSLICE_BYTES=$sb
    run c2sys_sb${sb}_$rep config2 STRAGGLAR_SUBSLICE_BYTES=$sb STRAGGLAR_SYS_SCOPE=1
    run c3_sb${sb}_$rep config3_1GiB STRAGGLAR_SUBSLICE_BYTES=$sb
  done
done
