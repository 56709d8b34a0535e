"""LL vs regular Phase B: device time of the fused single-call AllReduce."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_23523_b200 import stragglar as S  # noqa: E402

torch.cuda.set_device(0)
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def dev_time(fn, iters=20):
    fn()
    torch.cuda.synchronize()
    torch.cuda._sleep(6_000_000)
    a, b = ev(), ev()
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) * 1e3 / iters, 2)


out = {}
for n in (2, 8):
    for count in (1024, 16384, 131072, 458752):
        bufs = [torch.randn(count, device="cuda").to(torch.bfloat16) for _ in range(n)]
        for ll in ("0", "262144"):
            os.environ["STRAGGLAR_LL_MAX_CHUNK"] = ll
            S.stragglar_team_init(n, 0)                # knobs are read at init
            out[f"n{n}_c{count}_ll{ll}_fused"] = dev_time(lambda: S.stragglar_team_allreduce(bufs))
            out[f"n{n}_c{count}_ll{ll}_B"] = dev_time(lambda: (S.stragglar_team_reduce_scatter(bufs),
                                                               S.stragglar_team_complete(bufs)))
    assert S.stragglar_team_check_error() == 0
print(json.dumps(out, indent=1))
