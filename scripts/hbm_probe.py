"""HBM ceilings by access mix through torch ops: read-only, copy (1:1), write-only.

The 1 read : 4 writes mix (the direct completion's) is measured by scripts/hbm_mix.cu."""
import json
import torch

torch.cuda.set_device(0)
N = 1 << 30  # 1 Gi fp32 = 4 GiB
a = torch.empty(N, device="cuda")
b = torch.empty(N, device="cuda")
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def t(fn, bytes_moved, it=10):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(it):
        e0, e1 = ev(), ev()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    return round(bytes_moved / best / 1e9, 1)


res = {
    "write_only_fill_GBps": t(lambda: a.fill_(1.0), 4 * N),
    "copy_GBps": t(lambda: b.copy_(a), 8 * N),
    "read_only_sum_GBps": t(lambda: a.sum(), 4 * N),
}
print(json.dumps(res))
