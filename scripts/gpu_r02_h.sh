#!/bin/bash
# Lane-aware slice size sweep (n = 4, 8; bf16 1-64 MiB), config-5 bench, and the
# config-5 Phase-B trace at gpu and system scope.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02h}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; exit 1; }
for m in 0 32768 65536 131072; do
  STRAGGLAR_LANE_SLICE_MAX=$m timeout 900 python scripts/sweep.py --sizes-only --worlds 4,8 --max-log2-bytes 26 --iters 10 > gpurun_out/${T}_sweep_lsm$m.json 2> gpurun_out/${T}_sweep_lsm$m.err; echo "sweep lsm=$m rc=$?"
done
for m in 0 65536; do
  STRAGGLAR_LANE_SLICE_MAX=$m timeout 300 python bench.py --workload config5 --no-cpu --steps 30 --warmup 5 > gpurun_out/${T}_c5_lsm$m.json 2>/dev/null
  echo "c5 lsm=$m $(python -c "import json;d=json.load(open('gpurun_out/${T}_c5_lsm$m.json'));print(d['value'], d['T_post_stats_us']['median'], d['fused_call']['us'], d['T_phaseA_us'])" 2>&1 | tail -1)"
done
for sc in 0 1; do
  STRAGGLAR_SYS_SCOPE=$sc N=8 SIGMA=3 DTYPE=bfloat16 COUNT=524288 timeout 120 python scripts/trace_small.py > gpurun_out/${T}_trace_c5_sys$sc.json 2>&1; echo "trace sys=$sc rc=$?"
done
