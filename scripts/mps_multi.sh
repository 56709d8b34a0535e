#!/bin/bash
# Per-process mode, 8 ranks on one GPU running concurrently under MPS (each
# client limited to ~1/8 of the SMs so every rank's cooperative grid fits).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d && echo "mps started"
sleep 2
export CUDA_MPS_ACTIVE_THREAD_PERCENTAGE=${PCT:-12}
export STRAGGLAR_SLICES=${SLICES:-64} STRAGGLAR_TIMEOUT_MS=30000
N=${N:-8}
timeout 600 python -m torch.distributed.run --standalone --local-addr 127.0.0.1 --nproc-per-node $N bench.py --gpus $N --steps 5 --warmup 3 \
   --workload ${WL:-config2} > gpurun_out/mps_multi_$N.json 2> gpurun_out/mps_multi_$N.err
echo "bench rc=$?"
cat gpurun_out/mps_multi_$N.json
grep -iE "error|Timeout|illegal" gpurun_out/mps_multi_$N.err | head -5
echo quit | nvidia-cuda-mps-control
cat /tmp/mps_log/control.log 2>/dev/null | tail -3
