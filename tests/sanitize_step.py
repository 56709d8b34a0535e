"""Small team-mode calls for compute-sanitizer (memcheck / racecheck / synccheck):
both movers, n = 4 and 8, StragglAR + Ring + RHD + Broadcast, ragged count, checked vs the oracle;
then with small slice targets so every CTA covers several slices (sub-slices),
StragglAR fused and split (with the straggler delay), direct completion and the
NEXT-N3 baselines (RHD, Broadcast one launch and split)."""
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
    rhd = [b.clone() for b in bufs]
    bc = [b.clone() for b in bufs]
    S.stragglar_team_allreduce(bufs)
    S.stragglar_team_allreduce_ring(ring)
    S.stragglar_team_allreduce_rhd(rhd)          # NEXT N3 baselines
    S.stragglar_team_allreduce_bcast(bc)
    torch.cuda.synchronize()
    assert S.stragglar_team_check_error() == 0
    want, rwant = N.stragglar_allreduce(xs, sigma, "float32"), N.ring_allreduce(xs, "float32")
    hwant = N.rhd_allreduce(xs, "float32")
    for p in range(n):
        assert np.array_equal(bufs[p].cpu().numpy().view(np.uint32), want[p].view(np.uint32))
        assert np.array_equal(ring[p].cpu().numpy().view(np.uint32), rwant[p].view(np.uint32))
        assert np.array_equal(rhd[p].cpu().numpy().view(np.uint32), hwant[p].view(np.uint32))
        assert np.array_equal(bc[p].cpu().numpy().view(np.uint32), want[p].view(np.uint32))
os.environ["STRAGGLAR_SLICE_BYTES"] = "1024"
os.environ["STRAGGLAR_SUBSLICE_BYTES"] = "1024"
for n, sigma, count in [(4, 1, 200003), (8, 0, 400003)]:
    S.stragglar_team_init(n, sigma)
    xs = make_inputs(n, count, "float32", config=51)
    want = N.stragglar_allreduce(xs, sigma, "float32")
    for mode in ("fused", "split", "direct", "bcast", "rhd"):
        bufs = [torch.from_numpy(x).cuda() for x in xs]
        if mode == "fused":
            S.stragglar_team_allreduce(bufs)
        elif mode == "split":
            S.stragglar_team_reduce_scatter(bufs)
            S.stragglar_team_inject_delay(10_000)
            S.stragglar_team_complete(bufs)
        elif mode == "direct":
            S.stragglar_team_allreduce_direct(bufs)
        elif mode == "bcast":
            S.stragglar_team_bcast_precondition(bufs)
            S.stragglar_team_inject_delay(10_000)
            S.stragglar_team_bcast_complete(bufs)
        else:
            S.stragglar_team_allreduce_rhd(bufs)
        torch.cuda.synchronize()
        assert S.stragglar_team_check_error() == 0
        w = N.rhd_allreduce(xs, "float32") if mode == "rhd" else want
        for p in range(n):
            assert np.array_equal(bufs[p].cpu().numpy().view(np.uint32), w[p].view(np.uint32)), (mode, n, p)
print("sanitize step ok", os.environ.get("STRAGGLAR_MOVER", "default"))
