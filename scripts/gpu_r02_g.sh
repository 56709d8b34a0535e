#!/bin/bash
# Signal-thread A/B, then size sweeps (n = 8, bf16, 1-64 MiB) for the slice-size /
# op-lane defaults against the round-1 code (ab_old/).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02g}
TAG=$T bash scripts/gpu_r02_sig.sh
for v in "sb16k:STRAGGLAR_SLICE_BYTES=16384" "sb32k:STRAGGLAR_SLICE_BYTES=32768" "nolanes:STRAGGLAR_OP_LANES=1"; do
  name=${v%%:*}; envs=${v#*:}
  env $envs timeout 600 python scripts/sweep.py --sizes-only --worlds 8 --max-log2-bytes 26 --iters 10 > gpurun_out/${T}_sweep_$name.json 2> gpurun_out/${T}_sweep_$name.err; echo "sweep $name rc=$?"
done
(cd ab_old && timeout 600 python scripts/sweep.py --sizes-only --worlds 8 --max-log2-bytes 26 --iters 10 > ../gpurun_out/${T}_sweep_old.json 2> ../gpurun_out/${T}_sweep_old.err; echo "sweep old rc=$?")
