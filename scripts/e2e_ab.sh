#!/bin/bash
# A/B of the host-buffer pipeline knobs (piece size, copy streams) at config 2.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/e2e_ab
for pb in 4194304 8388608 16777216 33554432; do
  for ns in 1 2; do
    STRAGGLAR_E2E_PIECE_BYTES=$pb STRAGGLAR_E2E_STREAMS=$ns python bench.py --no-cpu --steps 5 --warmup 3 \
        > gpurun_out/e2e_ab/p${pb}_s$ns.json 2>/dev/null
    python - "$pb" "$ns" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/e2e_ab/p{sys.argv[1]}_s{sys.argv[2]}.json").read().strip().splitlines()[-1])
print(sys.argv[1], sys.argv[2], d["e2e"]["value"], d["e2e"]["pcie_floor_us"], d["e2e"]["frac_of_pcie_floor"])
PY
  done
done
