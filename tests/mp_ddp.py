"""DDP with the StragglAR comm hook vs DDP's default allreduce, n processes on
cuda:0 (gloo carries DDP's own traffic and the IPC blobs).  Launched by
tests/test_gpu_multiproc.py.  Exit 0 = gradients match the default hook and are
bitwise identical across ranks."""
import os
import sys

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def model():
    torch.manual_seed(1234)
    return torch.nn.Sequential(torch.nn.Linear(257, 513), torch.nn.GELU(), torch.nn.Linear(513, 129),
                               torch.nn.GELU(), torch.nn.Linear(129, 7)).cuda()


def worker(rank, world, sigma, port, mode, q):
    try:
        os.environ.setdefault("STRAGGLAR_SLICES", "8")
        os.environ.setdefault("STRAGGLAR_TIMEOUT_MS", "60000")
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        torch.cuda.set_device(rank % torch.cuda.device_count() if os.environ.get("STRAGGLAR_MP_SPREAD") else 0)   # one GPU per rank on a multi-GPU box
        from paper_2505_23523_b200.ddp import StragglarHookState, stragglar_hook
        from paper_2505_23523_b200.dist import ProcessComm

        comm = ProcessComm(sigma)
        ddp_s = torch.nn.parallel.DistributedDataParallel(model(), bucket_cap_mb=0.25)
        state = StragglarHookState(comm, mode=mode, expected_delay_ns=10_000_000)
        ddp_s.register_comm_hook(state, stragglar_hook)
        ddp_r = torch.nn.parallel.DistributedDataParallel(model(), bucket_cap_mb=0.25)
        g = torch.Generator().manual_seed(100 + rank)
        for step in range(3):
            x = torch.randn(64, 257, generator=g).cuda()
            for m in (ddp_s, ddp_r):
                m.zero_grad(set_to_none=True)
                m(x).square().mean().backward()
            torch.cuda.synchronize()
            gs = torch.cat([p.grad.flatten() for p in ddp_s.parameters()])
            gr = torch.cat([p.grad.flatten() for p in ddp_r.parameters()])
            err = ((gs - gr).abs().max() / gr.abs().max().clamp_min(1e-30)).item()
            allg = [torch.empty_like(gs.cpu()) for _ in range(world)]
            dist.all_gather(allg, gs.cpu())
            same = all(torch.equal(allg[0], t) for t in allg)
            if err > 1e-5 or not same:
                q.put((rank, f"step {step}: rel err {err:.3g}, ranks identical {same}"))
                return
        if mode == "auto":
            # bucket 0 behind a 10 ms expected delay -> StragglAR; later buckets the no-delay choice
            if not state.picks or any(a != "stragglar" for i, a in state.picks if i == 0):
                q.put((rank, f"auto picks {state.picks[:6]}"))
                return
        code = comm.lib.stragglar_check_error()
        state.close()
        comm.close()
        q.put((rank, "ok" if code == 0 else f"device error {code}"))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


if __name__ == "__main__":
    world, sigma, port, mode = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, world, sigma, port, mode, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    print(res)
    ok = all(v == "ok" for v in res.values())
    print("OK" if ok else "FAIL")
    sys.exit(0 if ok else 1)
