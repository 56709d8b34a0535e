#!/bin/bash
# ncu refresh on the final round-2 kernels: launch lists (profile_step.py, the bench command),
# full captures of the config-2 kernels (scripts/gpu_ncu.sh) and of the config-5 Phase B / fused call.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02y}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; exit 1; }
timeout 600 python bench.py --no-cpu --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$? $(python -c "import json;d=json.load(open('gpurun_out/${T}_bench.json'));print(d['value'], d['roofline']['frac'], d['e2e']['value'])")"
TAG=$T bash scripts/gpu_ncu.sh
for k in phaseB fused; do
  K=1; [ $k = fused ] && K=4
  PROFILE_COUNT=524288 PROFILE_DTYPE=bf16 PROFILE_SIGMA=3 timeout 600 ncu --set full --clock-control none --import-source on \
     --kernel-name-base demangled -k "regex:k_phase<.*\(int\)$K>" -s 2 -c 1 -o gpurun_out/${T}_c5_$k python scripts/profile_step.py > gpurun_out/${T}_c5_$k.log 2>&1; echo "c5 $k rc=$?"
done
NCU_SUMMARY_DIR=gpurun_out/ncu_summary_c5 python scripts/ncu_summary.py ${T}_c5 gpurun_out/${T}_c5_phaseB.ncu-rep gpurun_out/${T}_c5_fused.ncu-rep > /dev/null; echo "summary rc=$?"
rm -f gpurun_out/${T}_c5_fused.ncu-rep gpurun_out/${T}_c5_phaseB.ncu-rep
du -sh gpurun_out
