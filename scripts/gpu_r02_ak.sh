#!/bin/bash
# Signalling warp in Phase B (STRAGGLAR_SIGNALLER, variant lib_sig.so): parity, then A/B at GPU
# and system scope (team) and per process under MPS.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02ak}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; exit 1; }
V=$PWD/build/variants
STRAGGLAR_LIB=$V/lib_sig.so timeout 900 python -m pytest tests/test_gpu_team.py -x -q -k "medium or every_straggler or huge or subslices or system_scope or repeated or graph or full_size or knobs" > gpurun_out/${T}_pytest_sig.log 2>&1; echo "pytest team sig rc=$?"; tail -1 gpurun_out/${T}_pytest_sig.log
STRAGGLAR_LIB=$V/lib_sig.so timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q > gpurun_out/${T}_pytest_sig_mp.log 2>&1; echo "pytest mp sig rc=$?"; tail -1 gpurun_out/${T}_pytest_sig_mp.log
run() {
  local name=$1 wl=$2; shift 2
  env "$@" timeout 600 python bench.py --no-cpu --steps 20 --warmup 5 --workload $wl > gpurun_out/${T}_$name.json 2> gpurun_out/${T}_$name.err
  echo "$name rc=$? $(python -c "import json;d=json.load(open('gpurun_out/${T}_$name.json'));print(d['value'], d['T_post_stats_us']['median'], d['fused_call']['us'], d['ring_us'])" 2>&1 | tail -1)"
}
for rep in 1 2; do
  for v in default sig; do
    lib=$V/lib_$v.so; [ $v = default ] && lib=$PWD/paper_2505_23523_b200/libstragglar.so
    run c2_${v}_$rep config2 STRAGGLAR_LIB=$lib
    run c2sys_${v}_$rep config2 STRAGGLAR_LIB=$lib STRAGGLAR_SYS_SCOPE=1
    run c3sys_${v}_$rep config3_1GiB STRAGGLAR_LIB=$lib STRAGGLAR_SYS_SCOPE=1
  done
done
for v in default sig; do
  lib=$V/lib_$v.so; [ $v = default ] && lib=$PWD/paper_2505_23523_b200/libstragglar.so
  STRAGGLAR_LIB=$lib timeout 900 python bench.py --gpus 8 --mps --steps 20 --warmup 5 --no-cpu > gpurun_out/${T}_mps8_c2_$v.json 2> gpurun_out/${T}_mps8_c2_$v.err
  echo "mps8 c2 $v rc=$? $(python -c "
import json;d=json.loads(open('gpurun_out/${T}_mps8_c2_$v.json').read().strip().splitlines()[-1]);print(d['value'], d['T_phaseA_us'], {k:(v['T_post_us'], v['T_post_median_us']) for k,v in d['algorithms'].items()})" 2>&1 | tail -1)"
done
