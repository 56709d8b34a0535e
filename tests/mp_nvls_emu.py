"""NEXT N1(i) protocol check on one GPU: the NVLS kernel with its multicast
operations emulated through IPC peer pointers (stragglar_allreduce_nvls_emulated),
`world` processes sharing cuda:0 — repeated calls on fresh inputs, bit-exact vs
the oracle's canonical StragglAR result, every rank identical.  Launched by
tests/test_gpu_nvls.py.  Exit 0 = OK."""
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
        os.environ.setdefault("STRAGGLAR_SLICES", "8")
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2505_23523_b200 import stragglar as S
        from paper_2505_23523_b200.dist import ProcessComm
        from paper_2505_23523_b200.inputs import make_input

        comm = ProcessComm(sigma)
        buf = torch.zeros(count, dtype=TORCH[dtype], device="cuda")
        comm.register(buf)
        outs = []
        for call in range(3):
            x = make_input(count, dtype, rank, config=80 + call)
            xt = torch.from_numpy(x.view(np.int16) if dtype == "bfloat16" else x).view(TORCH[dtype])
            buf.copy_(xt.cuda())
            S.stragglar_allreduce_nvls_emulated(buf)
            outs.append(buf.cpu().view(torch.int16 if dtype == "bfloat16" else TORCH[dtype]).numpy().copy())
        torch.cuda.synchronize()
        code = S.stragglar_check_error()
        comm.close()
        q.put((rank, code, outs))
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
        r, code, outs = q.get(timeout=600)
        res[r] = (code, outs)
    for p in ps:
        p.join(timeout=60)
    bad = {r: c for r, (c, o) in res.items() if c != 0 or o is None}
    if bad:
        print("FAIL", bad)
        sys.exit(1)
    ok = True
    for call in range(3):
        want = N.stragglar_allreduce(make_inputs(world, count, dtype, config=80 + call), sigma, dtype)
        for r in range(world):
            got = res[r][1][call]
            w = want[r].view(np.int16) if dtype == "bfloat16" else want[r]
            if not np.array_equal(got.view(np.uint8), np.ascontiguousarray(w).view(np.uint8)):
                ok = False
                print(f"call {call} rank {r}: {int(np.count_nonzero(got != w))} elements differ")
    print("OK" if ok else "FAIL")
    sys.exit(0 if ok else 1)
