"""K0: the measured NVLink ceiling on a multi-GPU box —
peer copy bandwidth GPU 0 -> p and p -> 0 (copy engines, one direction at a
time) and GPU 0 receiving from all peers at once.  Prints one JSON line.
Needs >= 2 GPUs; on one GPU it prints {"skipped": ...}."""
import json
import sys

import torch


def timed_copy(dst, src, iters=10):
    dev = src.device if src.is_cuda else dst.device
    with torch.cuda.device(dev):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dst.copy_(src)
        torch.cuda.synchronize()
        s.record()
        for _ in range(iters):
            dst.copy_(src, non_blocking=True)
        e.record()
        torch.cuda.synchronize()
        return src.numel() * src.element_size() * iters / (s.elapsed_time(e) * 1e-3) / 1e9


def main():
    n = torch.cuda.device_count()
    if n < 2:
        print(json.dumps({"skipped": f"{n} GPU(s) visible; the NVLink probe needs >= 2"}))
        return
    nbytes = 256 << 20
    bufs = [torch.empty(nbytes // 4, device=f"cuda:{d}") for d in range(n)]
    out = {"gpus": n, "bytes": nbytes, "pairs": []}
    for p in range(1, n):
        tx = timed_copy(bufs[p], bufs[0])
        rx = timed_copy(bufs[0], bufs[p])
        out["pairs"].append({"peer": p, "gbps_0_to_p": round(tx, 1), "gbps_p_to_0": round(rx, 1)})
    # all peers write into GPU 0 at once (the straggler's ingress in a direct completion)
    dsts = [torch.empty(nbytes // 4, device="cuda:0") for _ in range(1, n)]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(device=f"cuda:{p}") for p in range(1, n)]
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.device(0):
        t0.record()
    for p, st, d in zip(range(1, n), streams, dsts):
        with torch.cuda.stream(st):
            st.wait_event(t0)
            for _ in range(5):
                d.copy_(bufs[p], non_blocking=True)
    for st in streams:
        with torch.cuda.device(0):
            torch.cuda.current_stream().wait_stream(st)
    with torch.cuda.device(0):
        t1.record()
    torch.cuda.synchronize()
    out["ingress_all_to_0_gbps"] = round((n - 1) * nbytes * 5 / (t0.elapsed_time(t1) * 1e-3) / 1e9, 1)
    print(json.dumps(out))


if __name__ == "__main__":
    sys.exit(main())
