#!/bin/bash
# Full round evidence in one gpurun call: GPU tests, smoke, bench, reference arm, ncu
# (scripts/gpu_final.sh), the size/delay sweep and the per-process mode under MPS.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r01g}
TAG=$TAG bash scripts/gpu_final.sh
timeout 1500 python scripts/sweep.py > gpurun_out/${TAG}_sweep.json 2> gpurun_out/${TAG}_sweep.err; echo "sweep rc=$?"
# each MPS client gets ~1/n of the SMs; slices per rank sized so every rank's grid fits
declare -A MPS_PCT=( [2]=50 [4]=25 [8]=12 ) MPS_SLICES=( [2]=128 [4]=64 [8]=64 )
for n in 2 4 8; do
  N=$n PCT=${MPS_PCT[$n]} SLICES=${MPS_SLICES[$n]} bash scripts/mps_multi.sh > gpurun_out/${TAG}_mps_$n.log 2>&1; echo "mps n=$n: $(grep 'bench rc' gpurun_out/${TAG}_mps_$n.log)"
  cp gpurun_out/mps_multi_$n.json gpurun_out/${TAG}_mps_$n.json 2>/dev/null
done
du -sh gpurun_out
