"""ranks whose layout knobs differ must not run with silently
different slice layouts.  Rank 1 sets another value of one knob (argv[2]=argv[3]:
the sub-slice size, the Phase-B unit order — a mixed order can deadlock —, or
the host pipeline's piece size); importing the handles must fail with
INVALID_ARG on every rank.  Launched by
tests/test_gpu_multiproc.py.  Exit 0 = behaved as specified."""
import os
import sys

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, port, q, knob, value):
    if rank == 1:
        os.environ[knob] = value
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=2)
    torch.cuda.set_device(0)
    from paper_2505_23523_b200 import stragglar as S
    from paper_2505_23523_b200.dist import ProcessComm

    try:
        ProcessComm(0)
        res = "accepted"
    except S.StragglarError as e:
        res = e.status
    dist.barrier()
    S.stragglar_finalize()
    q.put((rank, res))


if __name__ == "__main__":
    port = int(sys.argv[1])
    knob, value = (sys.argv[2], sys.argv[3]) if len(sys.argv) > 3 else ("STRAGGLAR_SUBSLICE_BYTES", "4096")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, port, q, knob, value)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    print(out)
    ok = out == {0: 1, 1: 1}
    print("OK" if ok else "FAIL")
    sys.exit(0 if ok else 1)
