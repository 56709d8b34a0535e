#!/bin/bash
# One gpurun call: smoke, GPU parity tests, multi-process probe, bench, ncu.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
OUT=gpurun_out
{
  nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
  which nvidia-cuda-mps-control || echo "no mps"
  nproc; lscpu | grep "Model name"; free -g | head -2
} > $OUT/env.txt 2>&1
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/rc.txt
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/rc.txt
timeout 240 python tests/mp_worker.py 2 1 100003 float32 29511 > $OUT/mp2.log 2>&1; echo "mp2 rc=$?" >> $OUT/rc.txt
timeout 600 python bench.py --steps 10 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/rc.txt
cat $OUT/rc.txt
