#!/bin/bash
# round evidence: GPU tests, smoke, bench (wall clock), reference arm, ncu launch lists + full captures
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r01d}
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
s=$(date +%s); python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$? wall=$(( $(date +%s) - s ))s"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_reference.json 2> gpurun_out/${TAG}_reference.err; echo "reference rc=$?"
TAG=$TAG bash scripts/gpu_ncu.sh
