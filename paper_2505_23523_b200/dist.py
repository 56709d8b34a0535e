"""Multi-process setup: one process per GPU, CUDA IPC handles exchanged over a
torch.distributed process group (NCCL on the GPU box, gloo in CPU tests).

torch.distributed is plumbing only: it carries the opaque handle blobs that
libstragglar.so exports; the collective itself never goes through it.
"""
from __future__ import annotations

from typing import List, Optional

import torch.distributed as dist


def all_gather_bytes(blob: bytes, group=None) -> bytes:
    """Concatenate every rank's blob in rank order (all blobs equal length)."""
    world = dist.get_world_size(group)
    out: List[Optional[bytes]] = [None] * world
    dist.all_gather_object(out, blob, group=group)
    if any(b is None or len(b) != len(blob) for b in out):
        raise RuntimeError("handle blobs of unequal size")
    return b"".join(out)  # type: ignore[arg-type]


class ProcessComm:
    """The per-process StragglAR communicator of this rank.

    ``lib`` is the binding module (``paper_2505_23523_b200.stragglar``); tests
    may pass a stand-in with the same function names.
    """

    def __init__(self, straggler_rank: int, group=None, lib=None):
        if lib is None:
            from . import stragglar as lib  # noqa: N813
        self.lib = lib
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.straggler = straggler_rank
        lib.stragglar_init(self.rank, self.world, straggler_rank)
        blobs = all_gather_bytes(lib.stragglar_export_handle(), group)
        lib.stragglar_import_handles(blobs, self.world)
        self.registered = []

    def register(self, tensor) -> None:
        """Collective: every rank registers its corresponding buffer."""
        blob = self.lib.stragglar_register_buffer(tensor)
        blobs = all_gather_bytes(blob, self.group)
        self.lib.stragglar_import_buffer(tensor, blobs, self.world)
        self.registered.append(tensor)

    def deregister(self, tensor) -> None:
        """Unmap the peers' copies of a registered buffer (every rank, before freeing it)."""
        self.lib.stragglar_deregister_buffer(tensor)
        self.registered = [t for t in self.registered if t is not tensor]

    def allreduce(self, tensor, stream=None) -> None:
        self.lib.stragglar_allreduce(tensor, stream)

    def allreduce_host(self, host_in, host_out, tensor, stream=None) -> None:
        """host_in -> tensor (registered) -> StragglAR -> host_out, pipelined in pieces."""
        self.lib.stragglar_allreduce_host(host_in, host_out, tensor, stream)

    def allreduce_ring(self, tensor, stream=None) -> None:
        self.lib.stragglar_allreduce_ring(tensor, stream)

    def allreduce_rhd(self, tensor, stream=None) -> None:
        self.lib.stragglar_allreduce_rhd(tensor, stream)

    def allreduce_bcast(self, tensor, stream=None) -> None:
        self.lib.stragglar_allreduce_bcast(tensor, stream)

    def close(self) -> None:
        self.lib.stragglar_finalize()
