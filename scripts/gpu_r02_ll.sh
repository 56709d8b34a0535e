#!/bin/bash
# Does the round-1 LL word protocol (ab_old/, removed in round 2) pay at SYSTEM
# scope, where every flag hand-off costs a MEMBAR.SYS?  Config 5 in team mode
# (gpu / sys scope, LL on / off) and per-process under MPS (8 ranks, sys scope).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02i}
cd ab_old
for sc in 0 1; do
  for ll in 0 262144; do
    STRAGGLAR_SYS_SCOPE=$sc STRAGGLAR_LL_MAX_CHUNK=$ll timeout 300 python bench.py --workload config5 --no-cpu --steps 30 --warmup 5 > ../gpurun_out/${T}_old_c5_sys${sc}_ll$ll.json 2>/dev/null
    echo "old c5 sys=$sc ll=$ll $(python -c "import json;d=json.load(open('../gpurun_out/${T}_old_c5_sys${sc}_ll$ll.json'));print(d['value'], d['fused_call']['us'])" 2>&1 | tail -1)"
  done
done
cd ..
for sc in 1; do
  STRAGGLAR_SYS_SCOPE=$sc timeout 300 python bench.py --workload config5 --no-cpu --steps 30 --warmup 5 > gpurun_out/${T}_new_c5_sys$sc.json 2>/dev/null
  echo "new c5 sys=$sc $(python -c "import json;d=json.load(open('gpurun_out/${T}_new_c5_sys$sc.json'));print(d['value'], d['fused_call']['us'])" 2>&1 | tail -1)"
done
