#!/bin/bash
# With sub-slice-major order + lifetime L2 hints (default now): stage ring / CTA shape and the
# sub-slice target re-tuned (scripts/build_variants.py --rs), two repetitions.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02ag}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; exit 1; }
V=$PWD/build/variants
run() {
  local name=$1 wl=$2; shift 2
  env "$@" timeout 600 python bench.py --no-cpu --steps 20 --warmup 5 --workload $wl > gpurun_out/${T}_$name.json 2> gpurun_out/${T}_$name.err
  echo "$name rc=$? $(python -c "import json;d=json.load(open('gpurun_out/${T}_$name.json'));print(d['value'], d['T_post_stats_us']['median'], d['T_phaseA_us'], d['fused_call']['us'], d['ring_us'], d['direct_completion']['T_post_us'], d['config']['slices_per_rank'])" 2>&1 | tail -1)"
}
for rep in 1 2; do
  for v in default s3_16k rs5 rs4 rs2; do
    lib=$V/lib_$v.so; [ $v = default ] && lib=$PWD/paper_2505_23523_b200/libstragglar.so
    run c2_${v}_$rep config2 STRAGGLAR_LIB=$lib
    run c3_${v}_$rep config3_1GiB STRAGGLAR_LIB=$lib
  done
  run c2sys_$rep config2 STRAGGLAR_SYS_SCOPE=1
done
timeout 1500 python -m pytest tests/test_gpu_team.py tests/test_gpu_multiproc.py -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${T}_pytest.log
