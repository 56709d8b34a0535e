#!/bin/bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02e}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; exit 1; }
nvcc -o /tmp/mc_selftest scripts/mc_selftest.cu -lcuda -Wno-deprecated-gpu-targets && /tmp/mc_selftest > gpurun_out/${T}_mc_selftest.txt 2>&1; echo "mc rc=$?"; grep -E "create-only|->" gpurun_out/${T}_mc_selftest.txt | tail -4
for sb in ${SBS:-16384 32768 65536}; do
  for lanes in 1 16; do
    STRAGGLAR_SLICE_BYTES=$sb STRAGGLAR_OP_LANES=$lanes timeout 300 python bench.py --workload config5 --no-cpu --steps 30 --warmup 5 > gpurun_out/${T}_c5_sb${sb}_l$lanes.json 2>/dev/null
    echo "c5 sb=$sb lanes=$lanes $(python -c "import json;d=json.load(open('gpurun_out/${T}_c5_sb${sb}_l$lanes.json'));print(d['value'], d['T_post_stats_us']['median'], d['fused_call']['us'], d['T_phaseA_us'], d['direct_completion']['T_post_us'])" 2>&1 | tail -1)"
  done
done
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$? $(python -c "import json;d=json.load(open('gpurun_out/${T}_bench.json'));print(d['value'], d['roofline']['frac'], d['fused_call']['us'])")"
