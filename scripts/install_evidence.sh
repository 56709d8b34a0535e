#!/bin/bash
# Copy one gpu_evidence.sh / gpu_final.sh run (gpurun_out/<TAG>_*) into the
# tracked profiles/r01/ and regenerate the sweep report.  Run here, after the
# gpurun call merged its gpurun_out/.
set -eu
cd "$(dirname "$0")/.."
TAG=${1:?usage: install_evidence.sh TAG}
P=profiles/r01
cp gpurun_out/${TAG}_bench.json $P/bench.json
cp gpurun_out/${TAG}_pytest.log $P/pytest_gpu.log
cp gpurun_out/${TAG}_smoke.log $P/smoke.log
cp gpurun_out/${TAG}_reference.json $P/reference_arm.json
cp gpurun_out/${TAG}_launches.csv $P/launches.csv
cp gpurun_out/${TAG}_bench_launches.csv $P/bench_launches.csv
cp gpurun_out/ncu_summary/${TAG}/ncu_summary.md $P/ncu_summary.md
cp gpurun_out/ncu_summary/${TAG}/ncu_summary.json $P/ncu_summary.json
sed "s#\"profiles/${TAG}/ncu_summary.json\"#\"profiles/r01/ncu_summary.json\"#" gpurun_out/ncu_summary/latest_traffic.json \
    > profiles/latest_traffic.json
if [ -f gpurun_out/${TAG}_sweep.json ]; then
  cp gpurun_out/${TAG}_sweep.json $P/sweep.json
  python scripts/sweep_report.py $P/sweep.json $P/sweep.md
fi
for n in 2 4 8; do
  [ -f gpurun_out/${TAG}_mps_$n.json ] && cp gpurun_out/${TAG}_mps_$n.json $P/mps/n${n}_sub1.json
done
echo "installed $TAG into $P"
