#!/bin/bash
# Round-2 ncu evidence on the final code: the bench command's launch list, full
# captures of the config-2 kernels (scripts/gpu_ncu.sh), and the latency-bound
# config-5 Phase B (op lanes).  One GPU, never a multi-rank command.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02_ncu_build.log 2>&1 || { echo build failed; exit 1; }
timeout 1500 python scripts/sweep.py > gpurun_out/r02_sweep.json 2> gpurun_out/r02_sweep.err; echo "sweep rc=$?"
TAG=r02 bash scripts/gpu_ncu.sh
PROFILE_COUNT=524288 PROFILE_DTYPE=bf16 PROFILE_SIGMA=3 timeout 600 ncu --set full --clock-control none --import-source on \
   --kernel-name-base demangled -k 'regex:k_phase<.*\(int\)1>' -s 2 -c 1 -o gpurun_out/r02_c5_phaseB python scripts/profile_step.py > gpurun_out/r02_c5_phaseB.log 2>&1; echo "c5 phaseB rc=$?"
PROFILE_COUNT=524288 PROFILE_DTYPE=bf16 PROFILE_SIGMA=3 timeout 600 ncu --set full --clock-control none --import-source on \
   --kernel-name-base demangled -k 'regex:k_phase<.*\(int\)4>' -s 2 -c 1 -o gpurun_out/r02_c5_fused python scripts/profile_step.py > gpurun_out/r02_c5_fused.log 2>&1; echo "c5 fused rc=$?"
NCU_SUMMARY_DIR=gpurun_out/ncu_summary python scripts/ncu_summary.py r02_c5 gpurun_out/r02_c5_phaseB.ncu-rep gpurun_out/r02_c5_fused.ncu-rep > /dev/null; echo "summary rc=$?"
rm -f gpurun_out/r02_c5_fused.ncu-rep
du -sh gpurun_out
