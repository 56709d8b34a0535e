"""One rank of the per-process (CUDA IPC) communicator, for running every rank
under compute-sanitizer directly (multiprocessing children are not followed):

    torchrun --standalone --local-addr 127.0.0.1 --nproc-per-node 2 --no-python \
        compute-sanitizer --tool memcheck --error-exitcode 9 python tests/mp_rank_sanitize.py

Ranks share cuda:0; gloo carries the IPC blobs.  Every algorithm of the
library runs once on a small ragged buffer (peer-mapped TMA loads/stores,
system-scope flags) and is checked against the oracle bit for bit.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    os.environ.setdefault("STRAGGLAR_TIMEOUT_MS", "300000")
    os.environ.setdefault("STRAGGLAR_SLICES", "4")
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(rank % torch.cuda.device_count() if os.environ.get("STRAGGLAR_MP_SPREAD") else 0)   # one GPU per rank on a multi-GPU box
    from oracle import numerics as N
    from paper_2505_23523_b200 import stragglar as S
    from paper_2505_23523_b200.dist import ProcessComm
    from paper_2505_23523_b200.inputs import make_input, make_inputs

    sigma, count, dtype = world - 1, 20001, "float32"
    comm = ProcessComm(sigma)
    x = torch.from_numpy(make_input(count, dtype, rank, config=9))
    algos = ["stragglar", "direct", "ring", "bcast"] + (["rhd"] if world & (world - 1) == 0 else [])
    bufs = {a: x.cuda() for a in algos}
    for b in bufs.values():
        comm.register(b)
    torch.cuda.synchronize()
    dist.barrier()
    comm.allreduce(bufs["stragglar"])
    S.stragglar_allreduce_direct(bufs["direct"])
    comm.allreduce_ring(bufs["ring"])
    comm.allreduce_bcast(bufs["bcast"])
    if "rhd" in bufs:
        comm.allreduce_rhd(bufs["rhd"])
    torch.cuda.synchronize()
    code = S.stragglar_check_error()
    xs = make_inputs(world, count, dtype, config=9)
    want = {"stragglar": N.stragglar_allreduce(xs, sigma, dtype), "direct": N.stragglar_allreduce(xs, sigma, dtype),
            "ring": N.ring_allreduce(xs, dtype), "bcast": N.broadcast_allreduce(xs, sigma, dtype)}
    if "rhd" in bufs:
        want["rhd"] = N.rhd_allreduce(xs, dtype)
    bad = [a for a in algos if not np.array_equal(bufs[a].cpu().numpy().view(np.uint32), want[a][rank].view(np.uint32))]
    dist.barrier()
    comm.close()
    dist.destroy_process_group()
    print(f"rank {rank}: device error {code}, mismatches {bad}")
    sys.exit(0 if code == 0 and not bad else 1)


if __name__ == "__main__":
    main()
