"""Time the direct completion (N1(ii)) and its HBM ceiling at config 2 in team mode.

Phase A, a masking delay, then `stragglar_team_complete_direct`, timed with CUDA events
on the launching stream (mean of the timed steps).  Also measures the HBM ceiling of
the direct completion's access mix (1 read : 4 writes) with a broadcast copy.  Honours
STRAGGLAR_LIB / STRAGGLAR_TEAM_SLICES / STRAGGLAR_MOVER for A/B runs.  Prints JSON."""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_23523_b200 import stragglar as S  # noqa: E402

torch.cuda.set_device(0)
n, sigma, count = 8, 0, 1 << 26
steps = int(os.environ.get("STEPS", "10"))
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
out = {}
if "--ceiling" in sys.argv:
    M = 1 << 28                                   # 1 GiB read, 4 GiB written
    a = torch.empty(M, device="cuda")
    big = torch.empty(M, 4, device="cuda")
    src = a.unsqueeze(1).expand(M, 4)
    big.copy_(src)
    best = 1e9
    for _ in range(10):
        e0, e1 = ev(), ev()
        e0.record()
        big.copy_(src)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    out["r1w4_broadcast_GBps"] = round(5 * 4 * M / best / 1e9, 1)
    del a, big, src
S.stragglar_team_init(n, sigma)
bufs = [torch.randn(count, device="cuda") for _ in range(n)]
C = (-(-count // (n - 1)) + 3) // 4 * 4 * 4
ts = []
for it in range(3 + steps):
    S.stragglar_team_reduce_scatter(bufs)
    S.stragglar_team_inject_delay(600_000)
    e0, e1 = ev(), ev()
    e0.record()
    S.stragglar_team_complete_direct(bufs)
    e1.record()
    torch.cuda.synchronize()
    if it >= 3:
        ts.append(e0.elapsed_time(e1) * 1e3)
assert S.stragglar_team_check_error() == 0
T = statistics.mean(ts)
out.update({"lib": os.environ.get("STRAGGLAR_LIB", "default"), "slices": S.stragglar_team_slices(),
            "mover": os.environ.get("STRAGGLAR_MOVER", "default"),
            "direct_us": round(T, 1), "direct_min_us": round(min(ts), 1),
            "hbm_GBps": round((n + 2) * (n - 1) * C / (T * 1e-6) / 1e9, 1)})
print(json.dumps(out))
