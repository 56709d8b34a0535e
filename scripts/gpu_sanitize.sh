#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export STRAGGLAR_TIMEOUT_MS=120000
for tool in memcheck racecheck synccheck; do
  for mover in tma lsu; do
    STRAGGLAR_MOVER=$mover timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tests/sanitize_step.py \
      > gpurun_out/sanitize_${tool}_${mover}.log 2>&1
    echo "$tool $mover rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize step ok' gpurun_out/sanitize_${tool}_${mover}.log | tr '\n' ' ')"
  done
done
