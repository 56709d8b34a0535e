#!/bin/bash
# ncu evidence for the team-mode kernels (one GPU; never a multi-rank command).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r01}
if [ -z "${SKIP_LISTS:-}" ]; then
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python scripts/profile_step.py > gpurun_out/${TAG}_launches.log 2>&1; echo "launches rc=$?"
# (demangled names read "k_phase<(int)1, (int)8, (int)1, (int)1>")
# the launch list of the bench command itself (cold-cache, serialised: shares, not absolutes)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench_under_ncu.log 2>&1; echo "bench launches rc=$?"
fi
# kernel-name regexes on the demangled names: k_phase<dtype, world, mover, KIND>
declare -A PAT=( [phaseB]='k_phase<.*\(int\)1>' [phaseA]='k_phase<.*\(int\)0>' [ring]='k_ring<' [direct]='k_phase<.*\(int\)3>'
                  [rhd]='k_rhd<' [bcast]='k_phase<.*\(int\)7>' [fused]='k_phase<.*\(int\)4>' )
for k in phaseB phaseA ring direct rhd bcast fused; do
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:${PAT[$k]}" -s 1 -c 1 \
      -o gpurun_out/${TAG}_$k python scripts/profile_step.py > gpurun_out/${TAG}_$k.log 2>&1; echo "$k rc=$?"
done
# summaries on the box (the .ncu-rep files are large); keep only the Phase-B report
NCU_SUMMARY_DIR=gpurun_out/ncu_summary python scripts/ncu_summary.py $TAG gpurun_out/${TAG}_phaseB.ncu-rep \
    gpurun_out/${TAG}_phaseA.ncu-rep gpurun_out/${TAG}_ring.ncu-rep gpurun_out/${TAG}_direct.ncu-rep \
    gpurun_out/${TAG}_rhd.ncu-rep gpurun_out/${TAG}_bcast.ncu-rep gpurun_out/${TAG}_fused.ncu-rep --traffic > /dev/null
rm -f gpurun_out/${TAG}_phaseA.ncu-rep gpurun_out/${TAG}_ring.ncu-rep gpurun_out/${TAG}_direct.ncu-rep \
    gpurun_out/${TAG}_rhd.ncu-rep gpurun_out/${TAG}_bcast.ncu-rep gpurun_out/${TAG}_fused.ncu-rep
du -sh gpurun_out
