#!/bin/bash
# System-scope release vs a CTA's TMA stream: drain / defer / signaller warp (scripts/fence_overlap.cu).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02w}
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fence_overlap scripts/fence_overlap.cu 2>/dev/null && \
  timeout 300 /tmp/fence_overlap > gpurun_out/${T}_fence_overlap.jsonl; echo "rc=$?"; cat gpurun_out/${T}_fence_overlap.jsonl
