"""Small team-mode calls for compute-sanitizer (memcheck / racecheck / synccheck):
both movers, n = 4 and 8, StragglAR + Ring, ragged count, checked vs the oracle;
then with small slice targets so every CTA covers several slices (sub-slices),
StragglAR fused and split (with the straggler delay) and direct completion."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import numerics as N  # noqa: E402
from paper_2505_23523_b200 import stragglar as S  # noqa: E402
from paper_2505_23523_b200.inputs import make_inputs  # noqa: E402

torch.cuda.set_device(0)
for n, sigma, count in [(4, 1, 40009), (8, 0, 100003)]:
    S.stragglar_team_init(n, sigma)
    xs = make_inputs(n, count, "float32", config=50)
    bufs = [torch.from_numpy(x).cuda() for x in xs]
    ring = [b.clone() for b in bufs]
    S.stragglar_team_allreduce(bufs)
    S.stragglar_team_allreduce_ring(ring)
    torch.cuda.synchronize()
    assert S.stragglar_team_check_error() == 0
    want, rwant = N.stragglar_allreduce(xs, sigma, "float32"), N.ring_allreduce(xs, "float32")
    for p in range(n):
        assert np.array_equal(bufs[p].cpu().numpy().view(np.uint32), want[p].view(np.uint32))
        assert np.array_equal(ring[p].cpu().numpy().view(np.uint32), rwant[p].view(np.uint32))
os.environ["STRAGGLAR_SLICE_BYTES"] = "1024"
os.environ["STRAGGLAR_SUBSLICE_BYTES"] = "1024"
for n, sigma, count in [(4, 1, 200003), (8, 0, 400003)]:
    S.stragglar_team_init(n, sigma)
    xs = make_inputs(n, count, "float32", config=51)
    want = N.stragglar_allreduce(xs, sigma, "float32")
    for mode in ("fused", "split", "direct"):
        bufs = [torch.from_numpy(x).cuda() for x in xs]
        if mode == "fused":
            S.stragglar_team_allreduce(bufs)
        elif mode == "split":
            S.stragglar_team_reduce_scatter(bufs)
            S.stragglar_team_inject_delay(10_000)
            S.stragglar_team_complete(bufs)
        else:
            S.stragglar_team_allreduce_direct(bufs)
        torch.cuda.synchronize()
        assert S.stragglar_team_check_error() == 0
        for p in range(n):
            assert np.array_equal(bufs[p].cpu().numpy().view(np.uint32), want[p].view(np.uint32)), (mode, n, p)
print("sanitize step ok", os.environ.get("STRAGGLAR_MOVER", "default"))
