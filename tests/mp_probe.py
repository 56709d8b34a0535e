"""K0 probes (stragglar_probe_copy / _pingpong) between 2 processes on cuda:0:
push and pull, TMA and 16-byte LSU, land exactly the right bytes in the right
segments; a short flag ping-pong completes and reports a positive time.
Launched by tests/test_gpu_multiproc.py.  Exit 0 = OK."""
import os
import sys

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, port, q):
    try:
        os.environ.setdefault("STRAGGLAR_SLICES", "8")
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=2)
        torch.cuda.set_device(0)
        from paper_2505_23523_b200 import stragglar as S
        from paper_2505_23523_b200.dist import ProcessComm

        comm = ProcessComm(1)
        pb = (1 << 20) + 4096
        buf = torch.zeros(2 * pb, dtype=torch.uint8, device="cuda")
        comm.register(buf)
        errs = []
        for mode in (S.PROBE_PUSH, S.PROBE_PULL, S.PROBE_TMA | S.PROBE_PUSH, S.PROBE_TMA | S.PROBE_PULL):
            g = torch.Generator(device="cuda").manual_seed(100 + rank + 10 * mode)
            buf.zero_()
            mine = torch.randint(0, 256, (pb,), generator=g, device="cuda", dtype=torch.uint8)
            buf[rank * pb:(rank + 1) * pb].copy_(mine)              # my own segment
            torch.cuda.synchronize()
            dist.barrier()
            S.stragglar_barrier()
            S.stragglar_probe_copy(buf, pb, mode, [1 - rank])
            torch.cuda.synchronize()
            dist.barrier()
            # after everyone's probe: segment p of every buffer holds rank p's data
            got = buf[(1 - rank) * pb:(2 - rank) * pb].cpu()
            theirs = [torch.zeros(pb, dtype=torch.uint8), torch.zeros(pb, dtype=torch.uint8)]
            dist.all_gather(theirs, mine.cpu())
            if not torch.equal(got, theirs[1 - rank]):
                errs.append(f"mode {mode}: segment {1 - rank} wrong")
        S.stragglar_barrier()
        S.stragglar_probe_pingpong(1 - rank, 5)
        us = S.stragglar_probe_pingpong_result()
        if not us > 0:
            errs.append(f"pingpong time {us}")
        comm.deregister(buf)
        code = S.stragglar_check_error()
        comm.close()
        q.put((rank, errs or ("ok" if code == 0 else f"device error {code}")))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


if __name__ == "__main__":
    port = int(sys.argv[1])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=600) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    print(out)
    ok = all(v == "ok" for v in out.values())
    print("OK" if ok else "FAIL")
    sys.exit(0 if ok else 1)
