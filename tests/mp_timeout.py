"""Watchdog check: rank 0 enters the collective, rank 1 never does.  The
device spin-waits must give up after STRAGGLAR_TIMEOUT_MS, report
ERR_TIMEOUT through stragglar_check_error, and the kernel must exit (no hang).
The error is sticky: the next call on the communicator fails with TIMEOUT
instead of launching on out-of-step flags.
Launched by tests/test_gpu_multiproc.py.  Exit 0 = behaved as specified."""
import os
import sys
import time

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, port, q):
    os.environ["STRAGGLAR_TIMEOUT_MS"] = "1500"
    os.environ["STRAGGLAR_SLICES"] = "4"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=2)
    torch.cuda.set_device(0)
    from paper_2505_23523_b200.dist import ProcessComm
    from paper_2505_23523_b200 import stragglar as S

    comm = ProcessComm(1)
    t = torch.ones(4096, device="cuda")
    comm.register(t)
    res = None
    if rank == 0:
        t0 = time.time()
        comm.allreduce(t)
        torch.cuda.synchronize()
        code, secs = S.stragglar_check_error(), time.time() - t0
        try:
            comm.allreduce(t)
            sticky = "no error"
        except S.StragglarError as e:
            sticky = e.status
        res = (code, secs, sticky)
    dist.barrier()
    comm.close()
    q.put((rank, res))


if __name__ == "__main__":
    port = int(sys.argv[1])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    code, secs, sticky = out[0]
    print(f"error code {code} after {secs:.2f} s; next call: {sticky}")
    ok = code == 1 and secs < 60 and sticky == 6
    print("OK" if ok else "FAIL")
    sys.exit(0 if ok else 1)
