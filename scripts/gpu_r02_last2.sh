#!/bin/bash
# Last check with the signalling warp on by default: smoke, the whole GPU suite, the default
# bench line, and the Phase-B ncu capture whose DRAM bytes the bench line reports.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02last2}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; exit 1; }
timeout 300 python __graft_entry__.py smoke > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${T}_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${T}_pytest.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$? $(python -c "import json;d=json.load(open('gpurun_out/${T}_bench.json'));r=d['roofline'];print(d['value'], r['frac'], r['traffic'], d['fused_call']['us'], d['ring_us'], d['direct_completion']['T_post_us'], d['e2e']['value'], d['gpu_launches'], d['clocks'])")"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:k_phase<.*\(int\)1>' -s 1 -c 1 -o gpurun_out/${T}_phaseB python scripts/profile_step.py > gpurun_out/${T}_phaseB.log 2>&1; echo "ncu phaseB rc=$?"
NCU_SUMMARY_DIR=gpurun_out/ncu_summary python scripts/ncu_summary.py $T gpurun_out/${T}_phaseB.ncu-rep --traffic; echo "summary rc=$?"
timeout 600 python bench.py --workload config5 --no-cpu > gpurun_out/${T}_c5.json 2>/dev/null; echo "c5 team $(python -c "import json;d=json.load(open('gpurun_out/${T}_c5.json'));print(d['value'], d['fused_call']['us'], d['ring_us'])")"
