"""A/B of the sub-slice count (STRAGGLAR_SUBSLICES) for Phase B, team mode.

For each message size and sub-slice cap: Phase A, a masking delay, then Phase B
(Algorithm 1), timed with CUDA events on the launching stream; prints one JSON
row per (size, sub) with the mean and median Phase-B time.  Sizes are bf16
(BASELINE configs[2]) at n = 8 plus config 2 (fp32, 256 MiB)."""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_23523_b200 import stragglar as S  # noqa: E402

torch.cuda.set_device(0)
n = 8
iters = int(os.environ.get("ITERS", "15"))
subs = [int(x) for x in os.environ.get("SUBS", "1,2,4,8").split(",")]
cases = [(torch.bfloat16, 1 << k) for k in (25, 26, 27, 28, 29, 30)] + [(torch.float32, 1 << 28)]
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
for dt, nbytes in cases:
    count = nbytes // (2 if dt == torch.bfloat16 else 4)
    bufs = [torch.randn(count, device="cuda").to(dt) for _ in range(n)]
    for m in subs:
        os.environ["STRAGGLAR_SUBSLICES"] = str(m)
        S.stragglar_team_init(n, 0)
        ts = []
        for it in range(3 + iters):
            S.stragglar_team_reduce_scatter(bufs)
            S.stragglar_team_inject_delay(int(3 * nbytes / 6.5e12 * 1e9) + 50_000)
            e0, e1 = ev(), ev()
            e0.record()
            S.stragglar_team_complete(bufs)
            e1.record()
            torch.cuda.synchronize()
            if it >= 3:
                ts.append(e0.elapsed_time(e1) * 1e3)
        assert S.stragglar_team_check_error() == 0
        print(json.dumps({"dtype": str(dt).split(".")[-1], "bytes": nbytes, "sub": m,
                          "T_post_us": round(statistics.mean(ts), 1), "median_us": round(statistics.median(ts), 1)}),
              flush=True)
    del bufs
