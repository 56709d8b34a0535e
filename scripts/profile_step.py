"""Minimal driver for ncu: config-2 team workload (n=8, 256 MiB fp32 per rank),
a few StragglAR steps (Phase A, delay, Phase B), Ring, direct completion and
the N3 baselines (RHD, Broadcast precondition + completion)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__  # noqa: E402

__graft_entry__.build()
from paper_2505_23523_b200 import stragglar as S  # noqa: E402

world, sigma = 8, int(os.environ.get("PROFILE_SIGMA", "0"))
count = int(os.environ.get("PROFILE_COUNT", str(1 << 26)))
dt = {"f32": torch.float32, "bf16": torch.bfloat16}[os.environ.get("PROFILE_DTYPE", "f32")]
steps = int(os.environ.get("PROFILE_STEPS", "3"))
torch.cuda.set_device(0)
g = torch.Generator(device="cuda").manual_seed(0)
bufs = [torch.randn(count, device="cuda", generator=g).to(dt) for _ in range(world)]
S.stragglar_team_init(world, sigma)
for _ in range(steps):
    S.stragglar_team_reduce_scatter(bufs)
    S.stragglar_team_inject_delay(10_000)
    S.stragglar_team_complete(bufs)
    S.stragglar_team_allreduce_ring(bufs)
    S.stragglar_team_reduce_scatter(bufs)
    S.stragglar_team_complete_direct(bufs)
    S.stragglar_team_allreduce(bufs)               # Phase A + B in one launch (KIND 4)
    S.stragglar_team_allreduce_rhd(bufs)           # NEXT N3 baselines
    S.stragglar_team_bcast_precondition(bufs)
    S.stragglar_team_bcast_complete(bufs)
torch.cuda.synchronize()
assert S.stragglar_team_check_error() == 0
print("profile step ok", S.stragglar_launch_count())
