"""Per-process (IPC) communicator exercised with every rank on cuda:0.

Launched by tests/test_gpu_multiproc.py (and usable by hand):
    python tests/mp_worker.py <world> <straggler> <count> <dtype> <port>
Each process is one rank; torch.distributed (gloo) only exchanges the CUDA
IPC blobs.  Ranks share one GPU, so their kernels time-slice unless MPS is
running; the protocol must still complete (correct by construction).
Exit code 0 = every rank's result equals the oracle bit for bit.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def mixed_lengths(count):
    return [count, count // 3, 17, count // 2 + 5, 4099, count]


def worker(rank, world, sigma, count, dtype, port, q):
    try:
        os.environ.setdefault("STRAGGLAR_TIMEOUT_MS", "60000")
        os.environ.setdefault("STRAGGLAR_SLICES", "8")
        os.environ.setdefault("STRAGGLAR_E2E_PIECE_BYTES", "40000")   # several pieces for the host entry point
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        torch.cuda.set_device(rank % torch.cuda.device_count() if os.environ.get("STRAGGLAR_MP_SPREAD") else 0)   # one GPU per rank on a multi-GPU box
        from paper_2505_23523_b200.dist import ProcessComm
        from paper_2505_23523_b200.inputs import make_input
        from paper_2505_23523_b200 import stragglar as S

        comm = ProcessComm(sigma)
        x = make_input(count, dtype, rank, config=7)
        tdt = {"float32": torch.float32, "int32": torch.int32, "bfloat16": torch.bfloat16}[dtype]
        t = torch.empty(count, dtype=tdt, device="cuda")
        ring = torch.empty(count, dtype=tdt, device="cuda")
        autos = [torch.empty(count, dtype=tdt, device="cuda") for _ in range(4)]
        base = {k: torch.empty(count, dtype=tdt, device="cuda") for k in ("rhd", "bcast", "mixed")}   # NEXT N3
        comm.register(t)
        comm.register(ring)
        for b in base.values():
            comm.register(b)
        for a in autos:
            comm.register(a)
        host = torch.from_numpy(x.view(np.int16) if dtype == "bfloat16" else x)
        t.view(host.dtype).copy_(host)
        ring.view(host.dtype).copy_(host)
        for a in list(autos) + list(base.values()):
            a.view(host.dtype).copy_(host)
        torch.cuda.synchronize()
        dist.barrier()
        S.stragglar_barrier()
        if rank == sigma:
            S.stragglar_inject_delay(200_000)
        comm.allreduce(t)
        ta, tk = S.stragglar_phase_times()          # in-kernel stamps of that call
        assert 0.0 <= ta <= tk < 60e6, (ta, tk)
        comm.allreduce_ring(ring)
        if world & (world - 1) == 0:
            comm.allreduce_rhd(base["rhd"])
        comm.allreduce_bcast(base["bcast"])
        # back-to-back StragglAR calls of different sizes on prefixes of one
        # buffer, no host sync: a fast rank's next call (another slice
        # layout) must not disturb a slow rank's current one
        for n_el in mixed_lengths(count):
            comm.allreduce(base["mixed"][:n_el])
        # NEXT row N2: selection for an expected delay (0 and 10 ms)
        used = [S.stragglar_allreduce_auto(autos[0], 0), S.stragglar_allreduce_auto(autos[1], 10_000_000)]
        S.stragglar_allreduce_direct(autos[2])     # NEXT row N1(ii): same result as the schedule
        used.append("stragglar")
        # end to end from pinned host memory, pipelined pieces, result back in host memory
        hin = host.clone().pin_memory()
        hout = torch.empty_like(hin).pin_memory()
        comm.allreduce_host(hin.view(tdt), hout.view(tdt), autos[3])
        torch.cuda.synchronize()
        code, where = S.stragglar_check_error_where(False)
        err = f"{code} at 0x{where:x}" if code else 0
        out = t.view(host.dtype).cpu().numpy()
        rout = ring.view(host.dtype).cpu().numpy()
        aout = [(u, a.view(host.dtype).cpu().numpy().tobytes()) for u, a in zip(used, autos[:3])]
        aout.append(("stragglar", hout.numpy().tobytes()))
        bout = {k: b.view(host.dtype).cpu().numpy().tobytes() for k, b in base.items()}
        dist.barrier()
        comm.close()
        q.put((rank, err, out.tobytes(), rout.tobytes(), (aout, bout)))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e), None, None, None))


def run(world, sigma, count, dtype, port):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=worker, args=(r, world, sigma, count, dtype, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, err, out, rout, ab = q.get(timeout=600)
        res[r] = (err, out, rout, ab)
    for p in procs:
        p.join(timeout=60)
    from oracle import numerics as N
    from paper_2505_23523_b200 import stragglar as S
    from paper_2505_23523_b200.inputs import make_inputs

    xs = make_inputs(world, count, dtype, config=7)
    want = N.stragglar_allreduce(xs, sigma, dtype)
    rwant = N.ring_allreduce(xs, dtype)
    bwant = {"bcast": N.broadcast_allreduce(xs, sigma, dtype)}
    state = [x.copy() for x in xs]
    for n_el in mixed_lengths(count):
        out = N.stragglar_allreduce([x[:n_el] for x in state], sigma, dtype)
        for r in range(world):
            state[r][:n_el] = out[r]
    bwant["mixed"] = state
    if world & (world - 1) == 0:
        bwant["rhd"] = N.rhd_allreduce(xs, dtype)
    ok = True
    for r in range(world):
        err, out, rout, ab = res[r]
        if out is None or err:
            print(f"rank {r}: error {err}")
            ok = False
            continue
        aout, bout = ab
        for k, w in bwant.items():
            if bout[k] != w[r].tobytes():
                print(f"rank {r}: {k} baseline result differs from the oracle")
                ok = False
        if out != want[r].tobytes():
            print(f"rank {r}: stragglar result differs from the oracle")
            ok = False
        if rout != rwant[r].tobytes():
            print(f"rank {r}: ring result differs from the oracle")
            ok = False
        for used, b in aout:
            w = {"stragglar": want, "ring": rwant}.get(used) or N.rhd_allreduce(xs, dtype)
            if b != w[r].tobytes():
                print(f"rank {r}: auto ({used}) result differs from the oracle")
                ok = False
        esz = 2 if dtype == "bfloat16" else 4
        for (used, _), d in zip(aout[:2], (0.0, 10e-3)):
            if used != S.stragglar_select_algorithm(world, count * esz, d, 3e-6, 1 / 770e9)[0]:
                print(f"rank {r}: auto picked {used}, not the cost model's choice for delay {d}")
                ok = False
    return ok


if __name__ == "__main__":
    w, s, c, d, port = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], int(sys.argv[5])
    ok = run(w, s, c, d, port)
    print("OK" if ok else "FAIL")
    sys.exit(0 if ok else 1)
