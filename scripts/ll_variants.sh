#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python scripts/ll_probe.py > gpurun_out/llv_default.json 2>&1
for lib in build/variants/lib_ll_*.so; do
  name=$(basename $lib .so)
  STRAGGLAR_LIB=$PWD/$lib python scripts/ll_probe.py > gpurun_out/llv_$name.json 2>&1; echo "$name rc=$?"
done
