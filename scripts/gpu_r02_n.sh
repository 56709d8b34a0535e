#!/bin/bash
# Epoch ticket drawn at start / consumed at exit vs bump at start (libstragglar_startbump.so);
# the direct completion's TMA mix ceiling; parity.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02n}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_mix scripts/tma_mix.cu && /tmp/tma_mix > gpurun_out/${T}_tma_mix.jsonl; echo "tma_mix rc=$?"; cat gpurun_out/${T}_tma_mix.jsonl
L=$PWD/paper_2505_23523_b200
run() {
  local name=$1 wl=$2; shift 2
  env "$@" timeout 600 python bench.py --no-cpu --steps 20 --warmup 5 --workload $wl > gpurun_out/${T}_$name.json 2> gpurun_out/${T}_$name.err
  echo "$name rc=$? $(python -c "import json;d=json.load(open('gpurun_out/${T}_$name.json'));print(d['value'], d['T_post_stats_us']['median'], d['T_phaseA_us'], d['fused_call']['us'], d['ring_us'], d['direct_completion']['T_post_us'])" 2>&1 | tail -1)"
}
for rep in 1 2; do
  for v in ticket startbump; do
    lib=$L/libstragglar.so; [ $v != ticket ] && lib=$L/libstragglar_$v.so
    run c5_${v}_$rep config5 STRAGGLAR_LIB=$lib
    run c5sys_${v}_$rep config5 STRAGGLAR_LIB=$lib STRAGGLAR_SYS_SCOPE=1
    run c4_${v}_$rep config4 STRAGGLAR_LIB=$lib
    run c2_${v}_$rep config2 STRAGGLAR_LIB=$lib
  done
done
timeout 1800 python -m pytest tests/test_gpu_team.py tests/test_gpu_multiproc.py -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${T}_pytest.log
