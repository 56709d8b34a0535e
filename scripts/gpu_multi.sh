#!/bin/bash
# For a box with >= 2 GPUs (not available in round 1): the NVLink ceiling, the
# per-process parity tests with one GPU per rank, and the N-GPU bench lines.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-multi}
NG=$(python -c "import torch; print(torch.cuda.device_count())")
echo "GPUs: $NG"
python scripts/nvlink_probe.py > gpurun_out/${TAG}_nvlink.json 2>&1; cat gpurun_out/${TAG}_nvlink.json
for n in 2 4 8; do
  [ "$n" -gt "$NG" ] && continue
  STRAGGLAR_MP_SPREAD=1 timeout 600 python tests/mp_worker.py $n $((n - 1)) 1000003 float32 $((29600 + n)) \
      > gpurun_out/${TAG}_mp_$n.log 2>&1; echo "mp n=$n rc=$? $(tail -1 gpurun_out/${TAG}_mp_$n.log)"
  for wl in config2 config5; do
    timeout 900 python -m torch.distributed.run --standalone --local-addr 127.0.0.1 --nproc-per-node $n \
        bench.py --gpus $n --workload $wl > gpurun_out/${TAG}_bench_${wl}_$n.json 2> gpurun_out/${TAG}_bench_${wl}_$n.err
    echo "bench $wl n=$n rc=$?"; tail -c 400 gpurun_out/${TAG}_bench_${wl}_$n.json; echo
  done
done
