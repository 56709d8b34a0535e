"""Per-op timeline of a small-message Phase B (latency-bound regime) from the in-kernel trace.

n = 8, straggler 0, fp32, a few KB per chunk (one slice): for every rank and op, how long the
op waited for its flag (wait -> data) and how long its data movement + signal took
(data -> done), in ns.  Shows where a round's ~2.5 us goes at small sizes."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_23523_b200 import stragglar as S  # noqa: E402

n, sigma = int(os.environ.get("N", "8")), int(os.environ.get("SIGMA", "0"))
count = int(os.environ.get("COUNT", "4096"))
dt = {"float32": torch.float32, "bfloat16": torch.bfloat16}[os.environ.get("DTYPE", "float32")]
torch.cuda.set_device(0)
S.stragglar_team_init(n, sigma)
bufs = [torch.randn(count, device="cuda").to(dt) for _ in range(n)]
for _ in range(5):
    S.stragglar_team_allreduce(bufs)
S.stragglar_team_set_trace(True)
out = []
for rep in range(5):
    S.stragglar_team_reduce_scatter(bufs)
    S.stragglar_team_inject_delay(50_000)
    S.stragglar_team_complete(bufs)
    torch.cuda.synchronize()
    tr, NS = S.stragglar_team_read_trace()
    t0 = min(v for v in tr if v)
    rows = {}
    for p in range(n):
        ops = []
        for k in range(16):
            w, d, e = tr[((p * NS + 0) * 16 + k) * 3:((p * NS + 0) * 16 + k) * 3 + 3]
            if w and d and e:
                ops.append({"k": k, "start": w - t0, "wait": d - w, "move": e - d, "end": e - t0})
        rows[f"phys{p}"] = ops
    out.append({"rep": rep, "slices": NS, "end_ns": max(v for v in tr if v) - t0, "ranks": rows})
S.stragglar_team_set_trace(False)
assert S.stragglar_team_check_error() == 0
print(json.dumps(out[-1], indent=1))
print(json.dumps({"end_ns_per_rep": [o["end_ns"] for o in out]}))
