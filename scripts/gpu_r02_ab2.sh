#!/bin/bash
# Same-box A/B: round-1 code (ab_old/, built from 4fc125a) vs this tree with
# and without deferred hand-offs, gpu and system scope; config 5 latency.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02c}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; exit 1; }
run() {  # name, env..., -- args
  local name=$1; shift
  env "$@" timeout 600 python bench.py --no-cpu --steps 20 --warmup 5 ${WL:+--workload $WL} > gpurun_out/${T}_$name.json 2> gpurun_out/${T}_$name.err
  echo "$name rc=$? $(python -c "import json;d=json.load(open('gpurun_out/${T}_$name.json'));print(d['value'], d['T_phaseA_us'], d['fused_call']['us'], d['ring_us'], d['direct_completion']['T_post_us'])" 2>&1 | tail -1)"
}
for rep in 1 2; do
  (cd ab_old && timeout 600 python bench.py --no-cpu --steps 20 --warmup 5 > ../gpurun_out/${T}_old$rep.json 2> ../gpurun_out/${T}_old$rep.err; echo "old$rep rc=$? $(python -c "import json;d=json.load(open('../gpurun_out/${T}_old$rep.json'));print(d['value'], d['T_phaseA_us'], d['fused_call']['us'], d['ring_us'], d['direct_completion']['T_post_us'])" 2>&1 | tail -1)")
  run new_defer0_$rep STRAGGLAR_DEFER=0
  run new_defer1_$rep STRAGGLAR_DEFER=1
done
run sys1_sub16_defer1 STRAGGLAR_SYS_SCOPE=1 STRAGGLAR_DEFER=1
run sys1_sub16_defer0 STRAGGLAR_SYS_SCOPE=1 STRAGGLAR_DEFER=0
run sys1_sub1_defer1 STRAGGLAR_SYS_SCOPE=1 STRAGGLAR_SUBSLICES=1 STRAGGLAR_DEFER=1
WL=config5 run c5_defer1 STRAGGLAR_DEFER=1
WL=config5 run c5_defer0 STRAGGLAR_DEFER=0
(cd ab_old && timeout 600 python bench.py --no-cpu --steps 20 --warmup 5 --workload config5 > ../gpurun_out/${T}_c5_old.json 2>/dev/null; echo "c5 old $(python -c "import json;d=json.load(open('../gpurun_out/${T}_c5_old.json'));print(d['value'], d['fused_call']['us'])")")
if [ -n "${PYTEST_K:-}" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$PYTEST_K" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.log
fi
