#!/bin/bash
# L2 hints by data lifetime (Op::life; scripts/build_variants.py --life / --hint3) vs the default.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02ac}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; exit 1; }
V=$PWD/build/variants
run() {
  local name=$1 wl=$2; shift 2
  env "$@" timeout 600 python bench.py --no-cpu --steps 20 --warmup 5 --workload $wl > gpurun_out/${T}_$name.json 2> gpurun_out/${T}_$name.err
  echo "$name rc=$? $(python -c "import json;d=json.load(open('gpurun_out/${T}_$name.json'));print(d['value'], d['T_phaseA_us'], d['fused_call']['us'], d['ring_us'], d['baselines_N3']['rhd_us'])" 2>&1 | tail -1)"
}
for rep in 1 2; do
  for v in default life_ef life_none ld_none; do
    lib=$V/lib_$v.so; [ $v = default ] && lib=$PWD/paper_2505_23523_b200/libstragglar.so
    run c2_${v}_$rep config2 STRAGGLAR_LIB=$lib
    run c3_${v}_$rep config3_1GiB STRAGGLAR_LIB=$lib
  done
done
for v in life_ef life_none; do
  STRAGGLAR_LIB=$V/lib_$v.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none \
     --kernel-name-base demangled -k 'regex:k_phase<.*\(int\)1>' -s 1 -c 1 --csv python scripts/profile_step.py > gpurun_out/${T}_ncu_phaseB_$v.csv 2> gpurun_out/${T}_ncu_phaseB_$v.err
  echo "ncu $v rc=$?"; grep -E "dram__bytes|duration|hit_rate" gpurun_out/${T}_ncu_phaseB_$v.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
STRAGGLAR_LIB=$V/lib_life_ef.so timeout 900 python -m pytest tests/test_gpu_team.py -x -q -k "medium or every_straggler or huge or subslices" > gpurun_out/${T}_pytest_life.log 2>&1; echo "pytest life rc=$?"; tail -1 gpurun_out/${T}_pytest_life.log
