#!/bin/bash
# A/B of library variants built with -D knobs (epoch bump at kernel start vs
# exit; polling depth), config 5 / 4 / 2, gpu and system scope; then parity.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02j}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; exit 1; }
L=$PWD/paper_2505_23523_b200
run() {
  local name=$1 wl=$2; shift 2
  env "$@" timeout 600 python bench.py --no-cpu --steps 20 --warmup 5 --workload $wl > gpurun_out/${T}_$name.json 2> gpurun_out/${T}_$name.err
  echo "$name rc=$? $(python -c "import json;d=json.load(open('gpurun_out/${T}_$name.json'));print(d['value'], d['T_post_stats_us']['median'], d['T_phaseA_us'], d['fused_call']['us'], d['ring_us'], d['direct_completion']['T_post_us'])" 2>&1 | tail -1)"
}
for rep in 1 2; do
  for v in default exit poll4 poll2; do
    lib=$L/libstragglar.so; [ $v != default ] && lib=$L/libstragglar_$v.so
    run c5_${v}_$rep config5 STRAGGLAR_LIB=$lib
    run c5sys_${v}_$rep config5 STRAGGLAR_LIB=$lib STRAGGLAR_SYS_SCOPE=1
  done
done
for v in default exit poll4; do
  lib=$L/libstragglar.so; [ $v != default ] && lib=$L/libstragglar_$v.so
  run c4_$v config4 STRAGGLAR_LIB=$lib
  run c2_$v config2 STRAGGLAR_LIB=$lib
done
timeout 1800 python -m pytest tests -m gpu -x -q -k "not sanitizer" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${T}_pytest.log
