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
    def __init__(self, comm, use_direct: bool = False):
        self.comm = comm
        self.use_direct = use_direct
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
    if state.use_direct:
        state.comm.lib.stragglar_allreduce_direct(buf)
    else:
        state.comm.allreduce(buf)
    fut: torch.futures.Future[torch.Tensor] = torch.futures.Future()
    fut.set_result(buf)
    return fut
