#!/bin/bash
# Phase B unit order: op by op (default) vs sub-slice by sub-slice (STRAGGLAR_SUB_MAJOR=1):
# parity with the new order, team config 2 / 1 GiB bf16 / config 4 at GPU and system scope,
# MPS n = 8, and the Phase-B DRAM traffic of each order under ncu.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02z}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; exit 1; }
STRAGGLAR_SUB_MAJOR=1 timeout 1500 python -m pytest tests/test_gpu_team.py tests/test_gpu_multiproc.py -x -q > gpurun_out/${T}_pytest_sm1.log 2>&1; echo "pytest sub_major rc=$?"; tail -2 gpurun_out/${T}_pytest_sm1.log
run() {
  local name=$1 wl=$2; shift 2
  env "$@" timeout 600 python bench.py --no-cpu --steps 20 --warmup 5 --workload $wl > gpurun_out/${T}_$name.json 2> gpurun_out/${T}_$name.err
  echo "$name rc=$? $(python -c "import json;d=json.load(open('gpurun_out/${T}_$name.json'));print(d['value'], d['T_post_stats_us']['median'], d['T_phaseA_us'], d['fused_call']['us'], d['ring_us'])" 2>&1 | tail -1)"
}
for rep in 1 2; do
  for m in 0 1; do
    run c2_sm${m}_$rep config2 STRAGGLAR_SUB_MAJOR=$m
    run c2sys_sm${m}_$rep config2 STRAGGLAR_SUB_MAJOR=$m STRAGGLAR_SYS_SCOPE=1
    run c3_sm${m}_$rep config3_1GiB STRAGGLAR_SUB_MAJOR=$m
    run c4_sm${m}_$rep config4 STRAGGLAR_SUB_MAJOR=$m
  done
done
for m in 0 1; do
  STRAGGLAR_SUB_MAJOR=$m timeout 900 python bench.py --gpus 8 --mps --steps 20 --warmup 5 --no-cpu > gpurun_out/${T}_mps8_c2_sm$m.json 2> gpurun_out/${T}_mps8_c2_sm$m.err
  echo "mps8 c2 sm=$m rc=$? $(python -c "
import json;d=json.loads(open('gpurun_out/${T}_mps8_c2_sm$m.json').read().strip().splitlines()[-1]);print(d['value'], d['T_phaseA_us'], {k:(v['T_post_us'], v['T_post_median_us']) for k,v in d['algorithms'].items()})" 2>&1 | tail -1)"
  STRAGGLAR_SUB_MAJOR=$m timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none \
     --kernel-name-base demangled -k 'regex:k_phase<.*\(int\)1>' -s 1 -c 2 --csv python scripts/profile_step.py > gpurun_out/${T}_ncu_phaseB_sm$m.csv 2> gpurun_out/${T}_ncu_phaseB_sm$m.err
  echo "ncu sm=$m rc=$?"; grep -E "dram__bytes|duration|hit_rate" gpurun_out/${T}_ncu_phaseB_sm$m.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' | head -8
done
