#!/bin/bash
# Flag-hop cost by scope (one GPU), then the per-process path self-launched as
# N ranks sharing the GPU under MPS: config 2 at N = 2, 4, 8 and config 5 at 8.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02k}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pp scripts/pingpong_scope.cu && /tmp/pp > gpurun_out/${T}_pingpong_scope.jsonl; echo "pp rc=$?"; cat gpurun_out/${T}_pingpong_scope.jsonl
for n in ${NS:-2 4 8}; do
  timeout 900 python bench.py --gpus $n --mps --steps ${STEPS:-20} --warmup 5 > gpurun_out/${T}_mps_c2_n$n.json 2> gpurun_out/${T}_mps_c2_n$n.err
  echo "mps c2 n=$n rc=$? $(python -c "
import json;d=json.loads(open('gpurun_out/${T}_mps_c2_n$n.json').read().strip().splitlines()[-1]);print(d['value'], {k:v['T_post_us'] for k,v in d['algorithms'].items()}, d['k0']['alpha_us'], d['shared_device'])" 2>&1 | tail -1)"
done
for sub in 16; do
  STRAGGLAR_SUBSLICES=$sub timeout 900 python bench.py --gpus 4 --mps --steps ${STEPS:-20} --warmup 5 > gpurun_out/${T}_mps_c2_n4_sub$sub.json 2> gpurun_out/${T}_mps_c2_n4_sub$sub.err
  echo "mps c2 n=4 sub=$sub rc=$? $(python -c "
import json;d=json.loads(open('gpurun_out/${T}_mps_c2_n4_sub$sub.json').read().strip().splitlines()[-1]);print(d['value'], {k:v['T_post_us'] for k,v in d['algorithms'].items()})" 2>&1 | tail -1)"
done
timeout 900 python bench.py --gpus 8 --mps --workload config5 --steps ${STEPS:-20} --warmup 5 > gpurun_out/${T}_mps_c5_n8.json 2> gpurun_out/${T}_mps_c5_n8.err
echo "mps c5 n=8 rc=$? $(python -c "
import json;d=json.loads(open('gpurun_out/${T}_mps_c5_n8.json').read().strip().splitlines()[-1]);print(d['value'], {k:v['T_post_us'] for k,v in d['algorithms'].items()})" 2>&1 | tail -1)"
