#!/bin/bash
# Full round evidence in one gpurun call: GPU tests, smoke, bench, reference arm, ncu
# (scripts/gpu_final.sh), the size/delay sweep and the per-process mode under MPS.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r01g}
TAG=$TAG bash scripts/gpu_final.sh
timeout 1500 python scripts/sweep.py > gpurun_out/${TAG}_sweep.json 2> gpurun_out/${TAG}_sweep.err; echo "sweep rc=$?"
for n in 2 4 8; do
  N=$n SLICES=64 bash scripts/mps_multi.sh > gpurun_out/${TAG}_mps_$n.log 2>&1; echo "mps n=$n: $(grep 'bench rc' gpurun_out/${TAG}_mps_$n.log)"
  cp gpurun_out/mps_multi_$n.json gpurun_out/${TAG}_mps_$n.json 2>/dev/null
done
du -sh gpurun_out
