"""Host-buffer pipeline A/B, interleaved in one process: equal 8 MiB pieces vs pieces ramped at
both ends (STRAGGLAR_E2E_RAMP), config 2 (n = 8 team, 256 MiB fp32 per rank), plus the PCIe
floor (the same H2D + D2H bytes as concurrent plain copies).  Wall-clock per synchronous call."""
import json
import os
import statistics
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_23523_b200 import stragglar as S  # noqa: E402

n, count = 8, 1 << 26
torch.cuda.set_device(0)
bufs = [torch.empty(count, device="cuda") for _ in range(n)]
hin = [torch.randn(count).pin_memory() for _ in range(n)]
hout = [torch.empty(count).pin_memory() for _ in range(n)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def floor_once():
    torch.cuda.synchronize()
    t = time.perf_counter()
    with torch.cuda.stream(s1):
        for p in range(n):
            bufs[p].copy_(hin[p], non_blocking=True)
    with torch.cuda.stream(s2):
        for p in range(n):
            hout[p].copy_(bufs[(p + 1) % n], non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) * 1e6


res = {"ramp0": [], "ramp1": [], "floor": []}
for rnd in range(6):
    for r in (0, 1):
        os.environ["STRAGGLAR_E2E_RAMP"] = str(r)
        S.stragglar_team_init(n, 0)
        S.stragglar_team_allreduce_host(hin, hout, bufs)   # warm
        for _ in range(4):
            t = time.perf_counter()
            S.stragglar_team_allreduce_host(hin, hout, bufs)
            res[f"ramp{r}"].append((time.perf_counter() - t) * 1e6)
        S.stragglar_team_finalize()
        res["floor"].append(floor_once())
out = {k: {"median_us": round(statistics.median(v), 1), "min_us": round(min(v), 1), "mean_us": round(statistics.mean(v), 1),
           "n": len(v)} for k, v in res.items()}
print(json.dumps(out))
