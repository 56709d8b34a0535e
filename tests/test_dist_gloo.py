"""world_size-2 gloo test of the multi-process host logic (CPU only): the IPC
blob exchange that wires the per-process communicators together."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class FakeTensor:
    def __init__(self, ptr):
        self.ptr = ptr


class FakeLib:
    """Stand-in for the ctypes binding that records what the C ABI would see."""

    def __init__(self, rank):
        self.rank = rank
        self.calls = []

    def stragglar_init(self, rank, world, sigma):
        self.calls.append(("init", rank, world, sigma))

    def stragglar_export_handle(self):
        return bytes([self.rank]) * 80

    def stragglar_import_handles(self, blobs, world):
        self.calls.append(("import_handles", blobs, world))

    def stragglar_register_buffer(self, t):
        return bytes([100 + self.rank]) * 80 + t.ptr.to_bytes(8, "little")

    def stragglar_import_buffer(self, t, blobs, world):
        self.calls.append(("import_buffer", t.ptr, blobs, world))

    def stragglar_allreduce(self, t, stream=None):
        self.calls.append(("allreduce", t.ptr))

    def stragglar_allreduce_ring(self, t, stream=None):
        self.calls.append(("ring", t.ptr))

    def stragglar_allreduce_rhd(self, t, stream=None):
        self.calls.append(("rhd", t.ptr))

    def stragglar_allreduce_bcast(self, t, stream=None):
        self.calls.append(("bcast", t.ptr))

    def stragglar_finalize(self):
        self.calls.append(("finalize",))


def _worker(rank, world, port, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    from paper_2505_23523_b200.dist import ProcessComm

    lib = FakeLib(rank)
    comm = ProcessComm(straggler_rank=1, lib=lib)
    comm.register(FakeTensor(1000 + rank))
    comm.allreduce(FakeTensor(1000 + rank))
    comm.allreduce_ring(FakeTensor(1000 + rank))
    comm.allreduce_rhd(FakeTensor(1000 + rank))
    comm.allreduce_bcast(FakeTensor(1000 + rank))
    comm.close()
    q.put((rank, lib.calls))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_handle_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=30)
        assert p.exitcode == 0
    want_handles = b"".join(bytes([r]) * 80 for r in range(world))
    want_bufs = b"".join(bytes([100 + r]) * 80 + (1000 + r).to_bytes(8, "little") for r in range(world))
    for r in range(world):
        calls = got[r]
        assert calls[0] == ("init", r, world, 1)
        assert calls[1] == ("import_handles", want_handles, world)
        assert calls[2] == ("import_buffer", 1000 + r, want_bufs, world)
        assert calls[3] == ("allreduce", 1000 + r)
        assert calls[4:7] == [("ring", 1000 + r), ("rhd", 1000 + r), ("bcast", 1000 + r)]
        assert calls[7] == ("finalize",)


class _FakeComm:
    """Stands in for ProcessComm: records the collective registrations."""

    def __init__(self, world=4):
        self.world = world
        self.group = None
        self.registered = []

    def register(self, t):
        self.registered.append(t.numel())

    def deregister(self, t):
        pass


def test_ddp_staging_grows_at_the_same_bucket_everywhere():
    """the DDP hook must enter the collective registration on every
    rank together.  The staging buffer's growth depends only on the bucket
    sizes (identical on every rank), never on the bucket's address."""
    import torch

    from paper_2505_23523_b200.ddp import StragglarHookState

    sizes = [1000, 600, 5000, 5000, 700, 9000, 100]
    seqs = []
    for seed in range(3):
        comm = _FakeComm()
        st = StragglarHookState(comm)
        torch.manual_seed(seed)
        for n in sizes:
            b = torch.empty(n + int(torch.randint(0, 3, ())) * 0)   # fresh allocation every time
            v = st.staging(b)
            assert v.numel() == n and v.dtype == b.dtype
        seqs.append(list(comm.registered))
    assert seqs[0] == seqs[1] == seqs[2]
    assert len(seqs[0]) == 3                     # grew at buckets 0, 2 and 5 only
    assert seqs[0][0] >= 1000 and seqs[0][1] >= 5000 and seqs[0][2] >= 9000


def _fd_worker(rank, world, port, q):
    import tempfile

    import torch.distributed as dist

    from paper_2505_23523_b200.dist import exchange_fds

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    f = tempfile.TemporaryFile()
    f.write(f"rank{rank}".encode())
    f.flush()
    mine = {"file": f.fileno(), "none": -1} if rank != 1 else {"none": -1}
    got = exchange_fds(mine)
    seen = {}
    for peer, fds in sorted(got.items()):
        for label, fd in fds.items():
            seen[(peer, label)] = os.pread(fd, 16, 0).decode()   # the offset is shared by every copy
            os.close(fd)
    dist.destroy_process_group()
    q.put((rank, seen))


@pytest.mark.parametrize("world", [2, 3])
def test_fd_exchange_over_unix_sockets(world):
    """The NVLS setup's descriptor exchange (SCM_RIGHTS over abstract UNIX
    sockets): every rank receives every other rank's labelled fds — here
    temporary files — and can read through them; -1 entries are not sent."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_fd_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=30)
    for r in range(world):
        want = {(p, "file"): f"rank{p}" for p in range(world) if p not in (r, 1)}
        assert out[r] == want
