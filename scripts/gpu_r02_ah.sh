#!/bin/bash
# Baselines' own unit order at system scope (op-major per process): MPS n = 2 / 4 / 8, parity.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02ah}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${T}_pytest.log
for n in 2 4 8; do
  timeout 900 python bench.py --gpus $n --mps --steps 20 --warmup 5 > gpurun_out/${T}_mps_c2_n$n.json 2> gpurun_out/${T}_mps_c2_n$n.err
  echo "mps c2 n=$n rc=$? $(python -c "
import json;d=json.loads(open('gpurun_out/${T}_mps_c2_n$n.json').read().strip().splitlines()[-1]);print(d['value'], d['T_phaseA_us'], {k:(v['T_post_us'], v['T_post_median_us']) for k,v in d['algorithms'].items()}, d['k0']['alpha_us'])" 2>&1 | tail -1)"
done
timeout 900 python bench.py --gpus 8 --mps --workload config5 --steps 20 --warmup 5 > gpurun_out/${T}_mps_c5_n8.json 2> gpurun_out/${T}_mps_c5_n8.err
echo "mps c5 n=8 rc=$? $(python -c "
import json;d=json.loads(open('gpurun_out/${T}_mps_c5_n8.json').read().strip().splitlines()[-1]);print(d['value'], {k:(v['T_post_us'], v['T_post_median_us']) for k,v in d['algorithms'].items()})" 2>&1 | tail -1)"
timeout 600 python bench.py --no-cpu > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$? $(python -c "import json;d=json.load(open('gpurun_out/${T}_bench.json'));print(d['value'], d['roofline']['frac'], d['roofline']['dram_frac'], d['fused_call']['us'], d['ring_us'], d['baselines_N3'])")"
