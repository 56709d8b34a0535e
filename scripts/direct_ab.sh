#!/bin/bash
# A/B the direct completion (N1(ii)) at config 2: ceiling, slices, mover, stage variants.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
P="timeout 300 python scripts/direct_probe.py"
$P --ceiling
for g in 74 56 37; do STRAGGLAR_TEAM_SLICES=$g $P; done
STRAGGLAR_MOVER=lsu $P
for lib in build/variants/lib_*.so; do STRAGGLAR_LIB=$PWD/$lib $P; done
