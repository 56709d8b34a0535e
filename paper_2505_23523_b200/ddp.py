"""PyTorch DistributedDataParallel communication hook running StragglAR.

PAPER.md P:735-742 (App. E) integrated StragglAR into data-parallel training
so that the gradient AllReduce of every bucket goes through it, with the
persistent straggler remapped once.  Here the same glue is a DDP comm hook:

    comm = ProcessComm(straggler_rank)          # paper_2505_23523_b200.dist
    ddp.register_comm_hook(StragglarHookState(comm), stragglar_hook)

Every bucket's flat gradient buffer is peer-mapped the first time it is seen
(a collective step: DDP presents buckets in the same order on every rank) and
reduced in place by the per-process communicator.  Like DDP's default
allreduce hook the gradients are divided by the world size (before the sum,
as DDP does).  The division is the only torch op in the hook; the reduction
runs in the library's kernels.
"""

import torch
import torch.distributed as dist


class StragglarHookState:
    """mode: "schedule" (StragglAR, Algorithm 1), "direct" (one-round direct
    completion, NEXT N1(ii)) or "auto": P:744-748 — only the first AllReduce of
    a backward pass meets the straggler (the later ones are synchronised by it),
    so bucket 0 runs the cost model's choice for `expected_delay_ns` and every
    later bucket its choice for no delay (RHD / Ring / StragglAR by size,
    stragglar_allreduce_auto)."""

    def __init__(self, comm, use_direct: bool = False, mode: str = None, expected_delay_ns: int = 0):
        self.comm = comm
        self.mode = mode or ("direct" if use_direct else "schedule")
        if self.mode not in ("schedule", "direct", "auto"):
            raise ValueError(f"unknown mode {self.mode}")
        self.expected_delay_ns = int(expected_delay_ns)
        self.picks: list = []        # "auto": (bucket index, algorithm) per call, for inspection
        self._registered: list = []  # (data_ptr, nbytes) of peer-mapped bucket buffers

    def _ensure_registered(self, buf: torch.Tensor) -> None:
        p, nb = buf.data_ptr(), buf.numel() * buf.element_size()
        for q, qb in self._registered:
            if q <= p and p + nb <= q + qb:
                return
        self.comm.register(buf)                 # collective: all ranks reach it in bucket order
        self._registered.append((p, nb))


def stragglar_hook(state: StragglarHookState, bucket: dist.GradBucket) -> torch.futures.Future[torch.Tensor]:
    buf = bucket.buffer()
    state._ensure_registered(buf)
    buf.div_(state.comm.world)
    if state.mode == "direct":
        state.comm.lib.stragglar_allreduce_direct(buf)
    elif state.mode == "auto":
        delay = state.expected_delay_ns if bucket.index() == 0 else 0
        state.picks.append((bucket.index(), state.comm.lib.stragglar_allreduce_auto(buf, delay)))
    else:
        state.comm.allreduce(buf)
    fut: torch.futures.Future[torch.Tensor] = torch.futures.Future()
    fut.set_result(buf)
    return fut
