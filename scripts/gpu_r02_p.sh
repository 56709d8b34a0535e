#!/bin/bash
# Sub-slice target size at SYSTEM scope: team config 2 / 1 GiB, and per process under MPS (n = 8).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02p}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; exit 1; }
run() {
  local name=$1 wl=$2; shift 2
  env "$@" timeout 600 python bench.py --no-cpu --steps 20 --warmup 5 --workload $wl > gpurun_out/${T}_$name.json 2> gpurun_out/${T}_$name.err
  echo "$name rc=$? $(python -c "import json;d=json.load(open('gpurun_out/${T}_$name.json'));print(d['value'], d['T_phaseA_us'], d['fused_call']['us'], d['ring_us'], d['direct_completion']['T_post_us'])" 2>&1 | tail -1)"
}
for rep in 1 2; do
  for sb in 131072 262144 524288; do
    run c2sys_sb${sb}_$rep config2 STRAGGLAR_SYS_SCOPE=1 STRAGGLAR_SUBSLICE_BYTES=$sb
    run c3sys_sb${sb}_$rep config3_1GiB STRAGGLAR_SYS_SCOPE=1 STRAGGLAR_SUBSLICE_BYTES=$sb
  done
  for sb in 131072 262144; do
    STRAGGLAR_SUBSLICE_BYTES=$sb timeout 900 python bench.py --gpus 8 --mps --steps 10 --warmup 3 --workload config3_1GiB --no-cpu > gpurun_out/${T}_mps8_c3_sb${sb}_$rep.json 2> gpurun_out/${T}_mps8_c3_sb${sb}_$rep.err
    echo "mps8 c3 sb=$sb rep=$rep rc=$? $(python -c "
import json;d=json.loads(open('gpurun_out/${T}_mps8_c3_sb${sb}_$rep.json').read().strip().splitlines()[-1]);print(d['value'], d['T_phaseA_us'], {k:v['T_post_us'] for k,v in d['algorithms'].items()})" 2>&1 | tail -1)"
  done
done
