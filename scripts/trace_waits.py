"""Where a Phase-B CTA's time goes at config 2 (team, n = 8, straggler 0, 256 MiB fp32): per
CTA, the sum over its (op, sub-slice) units of the time spent waiting for the unit's input
flag (trace: wait -> data) and moving + signalling (data -> done), and the CTA's span.
STRAGGLAR_SYS_SCOPE=1 for system-scope flags.  One JSON line."""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_23523_b200 import stragglar as S  # noqa: E402

n, sigma, count = 8, 0, 1 << 26
torch.cuda.set_device(0)
S.stragglar_team_init(n, sigma)
bufs = [torch.randn(count, device="cuda") for _ in range(n)]
for _ in range(3):
    S.stragglar_team_allreduce(bufs)
S.stragglar_team_set_trace(True)
out = []
for rep in range(3):
    S.stragglar_team_reduce_scatter(bufs)
    S.stragglar_team_inject_delay(600_000)
    S.stragglar_team_complete(bufs)
    torch.cuda.synchronize()
    assert S.stragglar_team_check_error() == 0
    tr, NS = S.stragglar_team_read_trace()
    G = 74
    sub = NS // G
    t0 = min(v for v in tr if v)
    waits, moves, spans, first_wait = [], [], [], []
    for p in range(n):
        for s in range(G):
            w_sum = m_sum = 0
            lo, hi = None, None
            fw = None
            for j in range(sub):
                v = s * sub + j
                for k in range(16):
                    b = ((p * NS + v) * 16 + k) * 3
                    w, d, e = tr[b:b + 3]
                    if not (w and d and e):
                        continue
                    w_sum += d - w
                    m_sum += e - d
                    lo = w if lo is None else min(lo, w)
                    hi = e if hi is None else max(hi, e)
            if lo is None:
                continue
            waits.append(w_sum / 1e3)
            moves.append(m_sum / 1e3)
            spans.append((hi - lo) / 1e3)
            first_wait.append((lo - t0) / 1e3)
    out.append({"rep": rep, "ctas": len(waits), "wait_us_median": statistics.median(waits),
                "move_us_median": statistics.median(moves), "span_us_median": statistics.median(spans),
                "span_us_max": max(spans), "wait_us_max": max(waits), "start_us_median": statistics.median(first_wait),
                "end_us": (max(v for v in tr if v) - t0) / 1e3})
S.stragglar_team_set_trace(False)
print(json.dumps({"sys_scope": os.environ.get("STRAGGLAR_SYS_SCOPE", "0"), "reps": out}))
