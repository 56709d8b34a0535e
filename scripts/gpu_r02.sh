#!/bin/bash
# Round-2 GPU pass: parity suite, the N=1 bench, and the per-process bench
# self-launched as N ranks sharing the one GPU (MPS and time-sliced).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02a}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_K:-} > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"
  tail -3 gpurun_out/${T}_pytest.log
fi
for n in ${NS:-2 4}; do
  timeout 900 python bench.py --gpus $n --mps --steps ${STEPS:-20} --warmup 5 ${WL:+--workload $WL} > gpurun_out/${T}_multi_mps_n$n.json 2> gpurun_out/${T}_multi_mps_n$n.err
  echo "bench mps n=$n rc=$?"; tail -c 600 gpurun_out/${T}_multi_mps_n$n.json; grep -iE "error|Traceback" gpurun_out/${T}_multi_mps_n$n.err | head -5
done
if [ "${TIMESLICED:-1}" = 1 ]; then
  timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --workload config1 > gpurun_out/${T}_multi_ts_n2.json 2> gpurun_out/${T}_multi_ts_n2.err
  echo "bench time-sliced n=2 rc=$?"; tail -c 400 gpurun_out/${T}_multi_ts_n2.json
fi
if [ "${BENCH1:-1}" = 1 ]; then
  timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
fi
