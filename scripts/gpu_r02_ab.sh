#!/bin/bash
# A/B runs of round-2 kernel changes (team mode, one B200): op lanes on the
# latency-bound config 5, flag scope x sub-slices on config 2, and the release
# cost probe.  Outputs under gpurun_out/${TAG}_*.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02ab}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; tail gpurun_out/${T}_build.log; exit 1; }
if [ "${FENCE:-1}" = 1 ]; then
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fence_probe scripts/fence_probe.cu && timeout 120 /tmp/fence_probe > gpurun_out/${T}_fence_probe.jsonl; echo "fence rc=$?"
fi
if [ -n "${PYTEST_K:-}" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$PYTEST_K" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.log
fi
for wl in ${WLS:-config5 config4}; do
  for lanes in ${LANES:-1 16}; do
    STRAGGLAR_OP_LANES=$lanes timeout 300 python bench.py --workload $wl --no-cpu --steps 30 --warmup 5 > gpurun_out/${T}_${wl}_lanes$lanes.json 2> gpurun_out/${T}_${wl}_lanes$lanes.err
    echo "$wl lanes=$lanes rc=$? $(python -c "import json;d=json.load(open('gpurun_out/${T}_${wl}_lanes$lanes.json'));print(d['value'], d['T_post_stats_us'], d['fused_call']['us'], d['ring_us'])" 2>&1 | tail -1)"
  done
done
for cfg in ${SCOPES:-"0 16" "1 16" "1 1" "0 1"}; do
  set -- $cfg
  STRAGGLAR_SYS_SCOPE=$1 STRAGGLAR_SUBSLICES=$2 timeout 600 python bench.py --no-cpu --steps 20 --warmup 5 > gpurun_out/${T}_scope$1_sub$2.json 2> gpurun_out/${T}_scope$1_sub$2.err
  echo "sys=$1 sub=$2 rc=$? $(python -c "import json;d=json.load(open('gpurun_out/${T}_scope$1_sub$2.json'));print(d['value'], d['T_phaseA_us'], d['fused_call']['us'], d['ring_us'], d['direct_completion']['T_post_us'])" 2>&1 | tail -1)"
done
