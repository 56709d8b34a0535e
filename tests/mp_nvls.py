"""NEXT N1(i) worker: `world` processes, one GPU each, NVLS arena set up
through ProcessComm.nvls_setup, StragglAR-NVLS AllReduce, checked against the
plain definition (oracle) within the north_star tolerance — int32 exact — and
every rank's result bitwise identical.  Launched by tests/test_gpu_nvls.py."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

TORCH = {"float32": torch.float32, "bfloat16": torch.bfloat16, "int32": torch.int32}


def worker(rank, world, sigma, count, dtype, port, q):
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        torch.cuda.set_device(rank)
        from paper_2505_23523_b200.dist import ProcessComm
        from paper_2505_23523_b200.inputs import make_input

        comm = ProcessComm(sigma)
        es = torch.tensor([], dtype=TORCH[dtype]).element_size()
        arena = comm.nvls_setup(count * es)
        x = make_input(count, dtype, rank, config=77)
        xt = torch.from_numpy(x.view(np.int16) if dtype == "bfloat16" else x)
        buf = arena[: count * es].view(TORCH[dtype])
        buf.copy_(xt.view(TORCH[dtype]).cuda())
        for _ in range(3):   # repeated calls on fresh inputs: epochs and arrival handshakes
            buf.copy_(xt.view(TORCH[dtype]).cuda())
            comm.allreduce_nvls(buf)
        torch.cuda.synchronize()
        code = comm.lib.stragglar_check_error()
        out = buf.cpu().view(torch.int16 if dtype == "bfloat16" else TORCH[dtype]).numpy().copy()
        comm.close()
        q.put((rank, code, out))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e), None))


if __name__ == "__main__":
    world, sigma, count, dtype, port = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], int(sys.argv[5])
    from oracle import numerics as N
    from paper_2505_23523_b200.inputs import make_inputs

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, world, sigma, count, dtype, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(world):
        r, code, out = q.get(timeout=600)
        res[r] = (code, out)
    for p in ps:
        p.join(timeout=60)
    bad = {r: c for r, (c, o) in res.items() if c != 0 or o is None}
    if bad:
        print("FAIL", bad)
        sys.exit(1)
    xs = make_inputs(world, count, dtype, config=77)
    want = N.plain_allreduce(xs, sigma, dtype)
    outs = [res[r][1] for r in range(world)]
    same = all(np.array_equal(outs[0], o) for o in outs)
    if dtype == "int32":
        ok = all(np.array_equal(o, want) for o in outs)
        err = 0.0
    else:
        got = outs[0].view(np.uint16) if dtype == "bfloat16" else outs[0]
        err = float(N.rel_error_vs_abs_sum(got, want, xs, dtype))
        ok = err <= (1e-2 if dtype == "bfloat16" else 1e-5)
    print(f"world={world} dtype={dtype} ranks identical {same} max rel err vs sum|x| {err:.3g}")
    print("OK" if (ok and same) else "FAIL")
    sys.exit(0 if ok and same else 1)
