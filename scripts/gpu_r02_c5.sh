#!/bin/bash
# Config-5 latency (team mode): slice size x op lanes; NVLS one-GPU self-test; full GPU suite.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02d}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; exit 1; }
timeout 300 python -m pytest tests/test_gpu_nvls.py -q > gpurun_out/${T}_nvls.log 2>&1; echo "nvls rc=$?"; tail -3 gpurun_out/${T}_nvls.log
for sb in ${SBS:-4096 8192 16384 32768}; do
  for lanes in 1 16; do
    STRAGGLAR_SLICE_BYTES=$sb STRAGGLAR_OP_LANES=$lanes timeout 300 python bench.py --workload config5 --no-cpu --steps 30 --warmup 5 > gpurun_out/${T}_c5_sb${sb}_l$lanes.json 2>/dev/null
    echo "c5 sb=$sb lanes=$lanes $(python -c "import json;d=json.load(open('gpurun_out/${T}_c5_sb${sb}_l$lanes.json'));print(d['value'], d['T_post_stats_us']['median'], d['fused_call']['us'], d['direct_completion']['T_post_us'], d['config']['slices_per_rank'])" 2>&1 | tail -1)"
  done
done
if [ "${FULL:-1}" = 1 ]; then
  timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.log
fi
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$? $(python -c "import json;d=json.load(open('gpurun_out/${T}_bench.json'));print(d['value'], d['roofline']['frac'])")"
