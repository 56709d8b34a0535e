#!/bin/bash
# Host-buffer pipeline with ramped first / last pieces (STRAGGLAR_E2E_RAMP) vs equal pieces; parity of the host entry points.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02x}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_team.py tests/test_gpu_multiproc.py -x -q -k "host or multiproc or proc" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${T}_pytest.log
for rep in 1 2 3; do
  for r in 0 1; do
    STRAGGLAR_E2E_RAMP=$r timeout 600 python bench.py --no-cpu --steps 20 --warmup 5 > gpurun_out/${T}_ramp${r}_$rep.json 2> gpurun_out/${T}_ramp${r}_$rep.err
    echo "ramp=$r rep=$rep rc=$? $(python -c "import json;d=json.load(open('gpurun_out/${T}_ramp${r}_$rep.json'));e=d['e2e'];print(d['value'], e['value'], e.get('frac_of_pcie_floor'), e.get('pcie_floor_us'))" 2>&1 | tail -1)"
  done
done
