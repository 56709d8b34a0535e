#!/bin/bash
# Final round-2 evidence on the committed code (sub-slice-major order, lifetime L2 hints):
# smoke, the whole GPU suite, the driver's default bench line, the reference arm, the
# per-process path under MPS, team config 5, the ncu refresh and the size / world / delay sweep.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02f2}
{
  nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv
  nproc; lscpu | grep "Model name"; python -c "import torch;print(torch.__version__, torch.cuda.nccl.version())"
} > gpurun_out/${T}_env.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; exit 1; }
timeout 300 python __graft_entry__.py smoke > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${T}_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$? $(python -c "import json;d=json.load(open('gpurun_out/${T}_bench.json'));print(d['value'], d['roofline']['frac'], d['fused_call']['us'], d['ring_us'], d['e2e']['value'], d['clocks'])")"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_reference.json 2> gpurun_out/${T}_reference.err; echo "reference rc=$? $(tail -c 200 gpurun_out/${T}_reference.json)"
for n in 2 4 8; do
  timeout 900 python bench.py --gpus $n --mps --steps 20 --warmup 5 > gpurun_out/${T}_mps_c2_n$n.json 2> gpurun_out/${T}_mps_c2_n$n.err
  echo "mps c2 n=$n rc=$? $(python -c "
import json;d=json.loads(open('gpurun_out/${T}_mps_c2_n$n.json').read().strip().splitlines()[-1]);print(d['value'], d['T_phaseA_us'], {k:(v['T_post_us'], v['T_post_median_us']) for k,v in d['algorithms'].items()}, d['k0']['alpha_us'])" 2>&1 | tail -1)"
done
timeout 900 python bench.py --gpus 8 --mps --workload config5 --steps 20 --warmup 5 > gpurun_out/${T}_mps_c5_n8.json 2> gpurun_out/${T}_mps_c5_n8.err
echo "mps c5 n=8 rc=$? $(python -c "
import json;d=json.loads(open('gpurun_out/${T}_mps_c5_n8.json').read().strip().splitlines()[-1]);print(d['value'], {k:(v['T_post_us'], v['T_post_median_us']) for k,v in d['algorithms'].items()})" 2>&1 | tail -1)"
timeout 600 python bench.py --workload config5 --no-cpu > gpurun_out/${T}_c5.json 2>/dev/null; echo "c5 team $(python -c "import json;d=json.load(open('gpurun_out/${T}_c5.json'));print(d['value'], d['fused_call']['us'], d['ring_us'])")"
TAG=$T bash scripts/gpu_ncu.sh
for k in phaseB fused; do
  K=1; [ $k = fused ] && K=4
  PROFILE_COUNT=524288 PROFILE_DTYPE=bf16 PROFILE_SIGMA=3 timeout 600 ncu --set full --clock-control none --import-source on \
     --kernel-name-base demangled -k "regex:k_phase<.*\(int\)$K>" -s 2 -c 1 -o gpurun_out/${T}_c5_$k python scripts/profile_step.py > gpurun_out/${T}_c5_$k.log 2>&1; echo "c5 $k rc=$?"
done
NCU_SUMMARY_DIR=gpurun_out/ncu_summary_c5 python scripts/ncu_summary.py ${T}_c5 gpurun_out/${T}_c5_phaseB.ncu-rep gpurun_out/${T}_c5_fused.ncu-rep > /dev/null; echo "summary rc=$?"
rm -f gpurun_out/${T}_c5_fused.ncu-rep gpurun_out/${T}_c5_phaseB.ncu-rep
timeout 1800 python scripts/sweep.py > gpurun_out/${T}_sweep.json 2> gpurun_out/${T}_sweep.err; echo "sweep rc=$?"
du -sh gpurun_out
