#!/bin/bash
# A/B: the release fence issued by thread 0 (libstragglar_sig0.so, built with
# -DSTRAGGLAR_SIGNAL_TID=0) vs by warp 1 (the default build), gpu / system scope.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02g}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; exit 1; }
run() {
  local name=$1; shift
  env "$@" timeout 600 python bench.py --no-cpu --steps 20 --warmup 5 ${WL:+--workload $WL} > gpurun_out/${T}_$name.json 2> gpurun_out/${T}_$name.err
  echo "$name rc=$? $(python -c "import json;d=json.load(open('gpurun_out/${T}_$name.json'));print(d['value'], d['T_phaseA_us'], d['fused_call']['us'], d['ring_us'], d['direct_completion']['T_post_us'])" 2>&1 | tail -1)"
}
for rep in 1 2; do
  run sig0_gpu_$rep STRAGGLAR_LIB=$PWD/paper_2505_23523_b200/libstragglar_sig0.so
  run sig32_gpu_$rep
  run sig0_sys_$rep STRAGGLAR_LIB=$PWD/paper_2505_23523_b200/libstragglar_sig0.so STRAGGLAR_SYS_SCOPE=1
  run sig32_sys_$rep STRAGGLAR_SYS_SCOPE=1
done
WL=config5 run c5_sig0 STRAGGLAR_LIB=$PWD/paper_2505_23523_b200/libstragglar_sig0.so
WL=config5 run c5_sig32
WL=config5 run c5_sig32_sys STRAGGLAR_SYS_SCOPE=1
