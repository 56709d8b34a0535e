#!/bin/bash
# round-end evidence: bench (timed wall clock), ncu launch lists + full captures
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r01c}
/usr/bin/time -v python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
grep -E "Elapsed|Maximum resident" gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_reference.json 2> gpurun_out/${TAG}_reference.err; echo "reference rc=$?"
TAG=$TAG bash scripts/gpu_ncu.sh
