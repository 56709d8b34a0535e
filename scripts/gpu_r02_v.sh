#!/bin/bash
# Deferred SEND hand-off (STRAGGLAR_DEFER_SEND) A/B at GPU and system scope, and two
# diagnostic builds that put half of a system-scope hand-off at GPU scope
# (release fence / acquire polls) to find which half costs.  Variant libraries are
# built on the CPU box into build/variants/ (scripts/build_variants.py --defer).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02v}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; exit 1; }
timeout 1800 python -m pytest tests/test_gpu_team.py tests/test_gpu_multiproc.py -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${T}_pytest.log
V=$PWD/build/variants
run() {
  local name=$1 wl=$2; shift 2
  env "$@" timeout 600 python bench.py --no-cpu --steps 20 --warmup 5 --workload $wl > gpurun_out/${T}_$name.json 2> gpurun_out/${T}_$name.err
  echo "$name rc=$? $(python -c "import json;d=json.load(open('gpurun_out/${T}_$name.json'));print(d['value'], d['T_post_stats_us']['median'], d['T_phaseA_us'], d['fused_call']['us'], d['ring_us'], d['direct_completion']['T_post_us'])" 2>&1 | tail -1)"
}
for rep in 1 2; do
  for v in nodefer defer; do
    lib=$V/lib_$v.so
    run c2_${v}_$rep config2 STRAGGLAR_LIB=$lib
    run c2sys_${v}_$rep config2 STRAGGLAR_LIB=$lib STRAGGLAR_SYS_SCOPE=1
    run c5sys_${v}_$rep config5 STRAGGLAR_LIB=$lib STRAGGLAR_SYS_SCOPE=1
    run c3sys_${v}_$rep config3_1GiB STRAGGLAR_LIB=$lib STRAGGLAR_SYS_SCOPE=1
  done
  for v in diag_fence_gpu diag_acq_gpu; do
    run c2sys_${v}_$rep config2 STRAGGLAR_LIB=$V/lib_$v.so STRAGGLAR_SYS_SCOPE=1
  done
done
for v in nodefer defer; do
  STRAGGLAR_LIB=$V/lib_$v.so timeout 900 python bench.py --gpus 8 --mps --steps 20 --warmup 5 --no-cpu > gpurun_out/${T}_mps8_c2_$v.json 2> gpurun_out/${T}_mps8_c2_$v.err
  echo "mps8 c2 $v rc=$? $(python -c "
import json;d=json.loads(open('gpurun_out/${T}_mps8_c2_$v.json').read().strip().splitlines()[-1]);print(d['value'], d['T_phaseA_us'], {k:v['T_post_us'] for k,v in d['algorithms'].items()})" 2>&1 | tail -1)"
done
