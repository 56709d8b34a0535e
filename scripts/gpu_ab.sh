#!/bin/bash
# parity for both movers + bench A/B + multi-process probes
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-ab}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest.log
for m in lsu tma; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --mover $m > gpurun_out/${TAG}_bench_$m.json 2> gpurun_out/${TAG}_bench_$m.err; echo "bench $m rc=$?"
done
timeout 300 python tests/mp_worker.py 8 0 1000003 float32 29533 > gpurun_out/${TAG}_mp8.log 2>&1; echo "mp8 rc=$?"
