"""Per-round timeline of Phase B (Algorithm 1) from the in-kernel trace.

Config 2 in team mode (n = 8, straggler 0, 256 MiB fp32): Phase A, masking delay,
then Phase B with tracing on.  For every round r: when its ops started moving data
(first / median), when they were signalled (median / last), and the HBM bytes they
moved, to see where Phase B's time goes (the rounds of Algorithm 1 move 4C, 6C, 10C,
16C x 4, 14C x 2 in team mode)."""
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
S.stragglar_team_reduce_scatter(bufs)
S.stragglar_team_inject_delay(600_000)
S.stragglar_team_complete(bufs)
torch.cuda.synchronize()
assert S.stragglar_team_check_error() == 0
tr, G = S.stragglar_team_read_trace()
S.stragglar_team_set_trace(False)

# physical <-> logical (straggler swapped with n-1) and every rank's op list in round order
phys = list(range(n))
phys[n - 1], phys[sigma] = sigma, n - 1
ops = {p: [] for p in range(n)}
for r in range(S.stragglar_schedule_rounds(n)):
    for src, dst, c, kind in S.stragglar_schedule_round(n, r):
        ops[phys[src]].append((r, c, kind))
C = -(-(-(-count // (n - 1))) // 4) * 4 * 4          # chunk bytes (16-byte rounded)
rounds = {}
t_min = min(v for v in tr if v)
for p in range(n):
    for s in range(G):
        for k, (r, c, kind) in enumerate(ops[p]):
            base = ((p * G + s) * 16 + k) * 3
            w, d, e = tr[base:base + 3]
            if not (w and d and e):
                continue
            rounds.setdefault(r, []).append((w - t_min, d - t_min, e - t_min, kind))
rows = []
for r in sorted(rounds):
    v = rounds[r]
    nbytes = 0
    for p in range(n):
        for (rr, c, kind) in ops[p]:
            if rr == r:
                nbytes += 2 * C if kind == 1 else 2 * C   # copy: read C + write C; exchange half: 2 reads + 2 writes of C/2
    starts = sorted(x[1] for x in v)
    ends = sorted(x[2] for x in v)
    span = (ends[-1] - starts[0]) / 1e3
    rows.append({"round": r, "ops": len(v) // G, "hbm_bytes": nbytes,
                 "data_start_first_us": round(starts[0] / 1e3, 1), "data_start_median_us": round(statistics.median(starts) / 1e3, 1),
                 "done_median_us": round(statistics.median(ends) / 1e3, 1), "done_last_us": round(ends[-1] / 1e3, 1),
                 "op_time_median_us": round(statistics.median(x[2] - x[1] for x in v) / 1e3, 1),
                 "span_GBps": round(nbytes / (span * 1e-6) / 1e9, 1) if span > 0 else None})
total = max(r["done_last_us"] for r in rows)
# per rank: for every op, median over slices of (wait began, data began, signalled)
per_rank = {}
for p in range(n):
    lst = []
    for k, (r, c, kind) in enumerate(ops[p]):
        w_, d_, e_ = [], [], []
        for s in range(G):
            base = ((p * G + s) * 16 + k) * 3
            w, d, e = tr[base:base + 3]
            if w and d and e:
                w_.append(w - t_min); d_.append(d - t_min); e_.append(e - t_min)
        if w_:
            lst.append({"op": k, "round": r, "chunk": c, "kind": "exch" if kind == 0 else "copy",
                        "wait_us": round(statistics.median(w_) / 1e3, 1), "data_us": round(statistics.median(d_) / 1e3, 1),
                        "done_us": round(statistics.median(e_) / 1e3, 1), "done_max_us": round(max(e_) / 1e3, 1)})
    per_rank[f"phys{p}"] = lst
out = {"G": G, "chunk_bytes": C, "phase_b_trace_span_us": total, "rounds": rows, "per_rank": per_rank}
print(json.dumps(out, indent=1))
