#!/bin/bash
# Sub-slice-major order everywhere (StragglAR Phase B, Ring, RHD; default on): parity, the
# baselines with each order, and the sub-slice target size re-tuned for the new order.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02aa}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; exit 1; }
timeout 1800 python -m pytest tests/test_gpu_team.py tests/test_gpu_multiproc.py tests/test_gpu_nvls.py -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${T}_pytest.log
run() {
  local name=$1 wl=$2; shift 2
  env "$@" timeout 600 python bench.py --no-cpu --steps 20 --warmup 5 --workload $wl > gpurun_out/${T}_$name.json 2> gpurun_out/${T}_$name.err
  echo "$name rc=$? $(python -c "import json;d=json.load(open('gpurun_out/${T}_$name.json'));print(d['value'], d['T_phaseA_us'], d['fused_call']['us'], d['ring_us'], d['baselines_N3']['rhd_us'], d['roofline']['frac'])" 2>&1 | tail -1)"
}
for rep in 1 2; do
  run c2_sm0_$rep config2 STRAGGLAR_SUB_MAJOR=0
  run c2_sm1_$rep config2
  run c3_sm0_$rep config3_1GiB STRAGGLAR_SUB_MAJOR=0
  run c3_sm1_$rep config3_1GiB
done
for sb in 32768 65536 262144; do
  run c2_sb${sb} config2 STRAGGLAR_SUBSLICE_BYTES=$sb
  run c3_sb${sb} config3_1GiB STRAGGLAR_SUBSLICE_BYTES=$sb
  run c2sys_sb${sb} config2 STRAGGLAR_SUBSLICE_BYTES=$sb STRAGGLAR_SYS_SCOPE=1
done
run c2sys_sb131072 config2 STRAGGLAR_SYS_SCOPE=1
timeout 1800 python scripts/sweep.py > gpurun_out/${T}_sweep.json 2> gpurun_out/${T}_sweep.err; echo "sweep rc=$?"
