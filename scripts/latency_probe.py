"""Device-side latency floor: launches are queued behind a 3 ms GPU spin
(torch.cuda._sleep) so event intervals measure device execution, not Python
and launch-API submission time."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__  # noqa: E402

__graft_entry__.build()
from paper_2505_23523_b200 import stragglar as S  # noqa: E402

torch.cuda.set_device(0)
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def dev_time(fn, iters=10):
    fn()
    torch.cuda.synchronize()
    torch.cuda._sleep(6_000_000)          # ~3 ms blocker: the CPU queues everything below meanwhile
    a, b = ev(), ev()
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) * 1e3 / iters, 2)


out = {}
x = torch.zeros(16, device="cuda")
out["torch_add_us"] = dev_time(lambda: x.add_(1))
S.stragglar_team_init(2, 1)
out["delay0_us"] = dev_time(lambda: S.stragglar_team_inject_delay(0))
VARIANTS = [("tma", "0", "16384"), ("lsu", "0", "16384")]
for mover, sysscope, slicebytes in VARIANTS:
    for n in [2, 4, 8]:
        os.environ["STRAGGLAR_MOVER"] = mover
        os.environ["STRAGGLAR_SYS_SCOPE"] = sysscope
        os.environ["STRAGGLAR_SLICE_BYTES"] = slicebytes
        S.stragglar_team_init(n, 0)
        g = f"sys{sysscope}_sb{slicebytes}"
        for count in [1024, 1 << 19, 1 << 22]:
            bufs = [torch.randn(count, device="cuda").to(torch.bfloat16) for _ in range(n)]
            ring = [b.clone() for b in bufs]
            key = f"{mover}_n{n}_G{g}_c{count}"
            out[key + "_AB"] = dev_time(lambda: (S.stragglar_team_reduce_scatter(bufs), S.stragglar_team_complete(bufs)))
            out[key + "_fused"] = dev_time(lambda: S.stragglar_team_allreduce(bufs))
            out[key + "_direct_fused"] = dev_time(lambda: S.stragglar_team_allreduce_direct(bufs))
            out[key + "_ring"] = dev_time(lambda: S.stragglar_team_allreduce_ring(ring))
        assert S.stragglar_team_check_error() == 0
for k in ["STRAGGLAR_SYS_SCOPE", "STRAGGLAR_SLICE_BYTES", "STRAGGLAR_MOVER"]:
    os.environ.pop(k, None)
print(json.dumps(out, indent=1))
