#!/bin/bash
# Phase A over a CTA's sub-slices as one range (STRAGGLAR_RS_WHOLE) vs slice by
# slice: team config 2 (gpu / system scope) and per-process under MPS (n = 8,
# sub-slices on), plus a parity subset with it on.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02m}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; exit 1; }
run() {
  local name=$1; shift
  env "$@" timeout 600 python bench.py --no-cpu --steps 20 --warmup 5 > gpurun_out/${T}_$name.json 2> gpurun_out/${T}_$name.err
  echo "$name rc=$? $(python -c "import json;d=json.load(open('gpurun_out/${T}_$name.json'));print(d['value'], d['T_phaseA_us'], d['fused_call']['us'], d['ring_us'], d['direct_completion']['T_post_us'])" 2>&1 | tail -1)"
}
for rep in 1 2; do
  for w in 0 1; do
    run whole${w}_gpu_$rep STRAGGLAR_RS_WHOLE=$w
    run whole${w}_sys_$rep STRAGGLAR_RS_WHOLE=$w STRAGGLAR_SYS_SCOPE=1
  done
done
for rep in 1 2; do
  for w in 0 1; do
    STRAGGLAR_RS_WHOLE=$w STRAGGLAR_SUBSLICES=16 timeout 900 python bench.py --gpus 8 --mps --steps 10 --warmup 3 --no-cpu > gpurun_out/${T}_mps8_whole${w}_$rep.json 2> gpurun_out/${T}_mps8_whole${w}_$rep.err
    echo "mps8 whole=$w rep=$rep rc=$? $(python -c "
import json;d=json.loads(open('gpurun_out/${T}_mps8_whole${w}_$rep.json').read().strip().splitlines()[-1]);print(d['value'], d['T_phaseA_us'], d['T_total_us'], {k:v['T_post_us'] for k,v in d['algorithms'].items()})" 2>&1 | tail -1)"
  done
done
STRAGGLAR_RS_WHOLE=1 timeout 1500 python -m pytest tests/test_gpu_team.py tests/test_gpu_multiproc.py -x -q -k "not sanitizer" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest whole=1 rc=$?"; tail -2 gpurun_out/${T}_pytest.log
