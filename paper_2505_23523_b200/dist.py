"""Multi-process setup: one process per GPU, CUDA IPC handles exchanged over a
torch.distributed process group (NCCL on the GPU box, gloo in CPU tests).

torch.distributed is plumbing only: it carries the opaque handle blobs that
libstragglar.so exports; the collective itself never goes through it.
"""
from __future__ import annotations

import json
import os
import secrets
import socket
from typing import Dict, List, Optional

import torch.distributed as dist


def all_gather_bytes(blob: bytes, group=None) -> bytes:
    """Concatenate every rank's blob in rank order (all blobs equal length)."""
    world = dist.get_world_size(group)
    out: List[Optional[bytes]] = [None] * world
    dist.all_gather_object(out, blob, group=group)
    if any(b is None or len(b) != len(blob) for b in out):
        raise RuntimeError("handle blobs of unequal size")
    return b"".join(out)  # type: ignore[arg-type]


def exchange_fds(fds: Dict[str, int], group=None) -> Dict[int, Dict[str, int]]:
    """Send this rank's labelled file descriptors (values < 0 are skipped) to
    every other rank of the node over abstract UNIX-domain sockets
    (SCM_RIGHTS); returns {peer rank: {label: received fd}}.  The caller owns
    (and closes) the received fds.  NVLS multicast objects and VMM arenas are
    shared this way: their POSIX handles are file descriptors, which a
    torch.distributed collective cannot carry."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    tok = [secrets.token_hex(8) if rank == 0 else None]
    dist.broadcast_object_list(tok, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    name = lambda r: f"\0stragglar-{tok[0]}-{r}"  # noqa: E731  (abstract namespace: no file to clean up)
    srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
    srv.bind(name(rank))
    srv.listen(world)
    dist.barrier(group)
    labels = [k for k, v in fds.items() if v is not None and v >= 0]
    payload = json.dumps({"from": rank, "labels": labels}).encode()
    for p in range(world):
        if p == rank:
            continue
        cl = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        cl.connect(name(p))
        socket.send_fds(cl, [payload], [fds[k] for k in labels])
        cl.close()
    got: Dict[int, Dict[str, int]] = {}
    for _ in range(world - 1):
        conn, _ = srv.accept()
        msg, rfds, _, _ = socket.recv_fds(conn, 4096, 16)
        info = json.loads(msg.decode())
        got[info["from"]] = dict(zip(info["labels"], rfds))
        conn.close()
    srv.close()
    dist.barrier(group)
    return got


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

    def nvls_setup(self, nbytes: int):
        """NEXT N1(i): allocate and bind this rank's NVLS arena (collective).
        Returns a uint8 CUDA tensor aliasing the arena; stragglar_allreduce_nvls
        reduces views of it in place."""
        try:
            fds, size = self.lib.stragglar_nvls_begin(nbytes)
            began = True
        except Exception as e:  # noqa: BLE001  (e.g. no multicast support): every rank must learn it
            began, err = False, e
        every = [None] * self.world
        dist.all_gather_object(every, began, group=self.group)
        if not all(every):
            if began:
                self.lib.stragglar_nvls_release()
            raise RuntimeError(f"NVLS arena setup failed on ranks {[r for r, v in enumerate(every) if not v]}"
                               + ("" if began else f": {err}"))
        got = exchange_fds({"mc_all": fds[0], "mc_ns": fds[1], "mem": fds[2]}, self.group)
        lowest_ns = 1 if self.straggler == 0 else 0
        mc_all = fds[0] if self.rank == 0 else got[0]["mc_all"]
        mc_ns = fds[1] if self.rank == lowest_ns else got.get(lowest_ns, {}).get("mc_ns", -1)
        sig_mem = got[self.straggler]["mem"] if self.rank != self.straggler else -1
        try:
            st = self.lib.stragglar_nvls_import(mc_all, mc_ns, sig_mem)
        finally:
            for peer in got.values():          # the library imported what it needs
                for fd in peer.values():
                    os.close(fd)
        # a bind waits for the whole team: bind only if every rank imported
        ok = [st == 0]
        every = [None] * self.world
        dist.all_gather_object(every, ok[0], group=self.group)
        if not all(every):
            if st == 0:
                self.lib.stragglar_nvls_release()
            raise RuntimeError(f"NVLS import failed on ranks {[r for r, v in enumerate(every) if not v]} (status {st})")
        ptr = self.lib.stragglar_nvls_bind()
        self.arena = self.lib.device_bytes(ptr, size)
        return self.arena

    def allreduce_nvls(self, tensor, stream=None) -> None:
        self.lib.stragglar_allreduce_nvls(tensor, stream)

    def close(self) -> None:
        self.arena = None
        self.lib.stragglar_finalize()
