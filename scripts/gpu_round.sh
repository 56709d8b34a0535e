#!/bin/bash
# parity (both movers) + bench (full contract) + ncu launch list + full captures
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r01b}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --mover lsu --no-cpu > gpurun_out/${TAG}_bench_lsu.json 2>> gpurun_out/${TAG}_bench.err; echo "bench lsu rc=$?"
TAG=$TAG bash scripts/gpu_ncu.sh
