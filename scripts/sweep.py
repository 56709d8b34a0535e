"""Message-size / world-size / delay sweeps on one B200 (single-device team).

BASELINE configs[2]: bf16, S = 2^20 .. 2^30 bytes, n in {2, 4, 8}, with and
without straggler delay; configs[3]/[4] points; and the delay sweep of
PAPER.md §4.2 (Fig. 4c analog) with the critical-delay condition
T_delay >= T_RS - max{T_B - T_SAR, 0}.

Writes one JSON document (rows) to stdout.  Timing: CUDA events on the
launching stream, warm-up first, buffers reused in place (values are not
checked here — parity is tests/test_gpu_team.py).
"""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__  # noqa: E402

__graft_entry__.build()
from paper_2505_23523_b200 import stragglar as S  # noqa: E402

ESZ = {torch.float32: 4, torch.bfloat16: 2}


def ev():
    return torch.cuda.Event(enable_timing=True)


def blocker():
    """Queue ~3 ms of GPU spin so the launches that follow are submitted while
    the GPU is busy: event intervals then measure device time, not Python /
    launch-API submission time (which is ~15 us per call through ctypes)."""
    torch.cuda._sleep(6_000_000)


def measure(n, sigma, count, dtype, iters, warm, delay_factor=1.25):
    S.stragglar_team_init(n, sigma)
    bufs = [torch.randn(count, device="cuda").to(dtype) for _ in range(n)]
    ring = [b.clone() for b in bufs]

    def run_split(d_ns, evs):
        evs[0].record()
        S.stragglar_team_reduce_scatter(bufs)
        evs[1].record()
        if d_ns is not None:
            S.stragglar_team_inject_delay(d_ns)
        evs[2].record()
        S.stragglar_team_complete(bufs)
        evs[3].record()

    for _ in range(warm):
        run_split(None, [ev() for _ in range(4)])
        S.stragglar_team_allreduce_ring(ring)
    torch.cuda.synchronize()
    # no delay: Phase A then Phase B back to back
    E = [[ev() for _ in range(4)] for _ in range(iters)]
    blocker()
    for e in E:
        run_split(None, e)
    torch.cuda.synchronize()
    T_A = statistics.median(e[0].elapsed_time(e[1]) * 1e3 for e in E)
    T_nod = statistics.median(e[0].elapsed_time(e[3]) * 1e3 for e in E)
    T_B_nod = statistics.median(e[2].elapsed_time(e[3]) * 1e3 for e in E)
    # masked delay
    D = int((delay_factor * T_A + 20.0) * 1e3)
    E = [[ev() for _ in range(4)] for _ in range(iters)]
    blocker()
    for e in E:
        run_split(D, e)
    torch.cuda.synchronize()
    T_tot = statistics.median(e[0].elapsed_time(e[3]) * 1e3 for e in E)
    T_post = statistics.median(e[2].elapsed_time(e[3]) * 1e3 for e in E)
    D_meas = statistics.median(e[0].elapsed_time(e[2]) * 1e3 for e in E)
    # ring
    R = [(ev(), ev()) for _ in range(iters)]
    blocker()
    for a, b in R:
        a.record()
        S.stragglar_team_allreduce_ring(ring)
        b.record()
    torch.cuda.synchronize()
    T_ring = statistics.median(a.elapsed_time(b) * 1e3 for a, b in R)
    # NEXT N3 baselines: RHD (whole AllReduce, like the Ring) and the Broadcast
    # baseline's post-arrival part (its precondition runs before the delay)
    T_rhd = None
    if n & (n - 1) == 0:
        for _ in range(warm):
            S.stragglar_team_allreduce_rhd(ring)
        R = [(ev(), ev()) for _ in range(iters)]
        blocker()
        for a, b in R:
            a.record()
            S.stragglar_team_allreduce_rhd(ring)
            b.record()
        torch.cuda.synchronize()
        T_rhd = statistics.median(a.elapsed_time(b) * 1e3 for a, b in R)
    B = [(ev(), ev()) for _ in range(iters + warm)]
    blocker()
    for a, b in B:
        S.stragglar_team_bcast_precondition(ring)
        S.stragglar_team_inject_delay(D)
        a.record()
        S.stragglar_team_bcast_complete(ring)
        b.record()
    torch.cuda.synchronize()
    T_bcast = statistics.median(a.elapsed_time(b) * 1e3 for a, b in B[warm:])
    assert S.stragglar_team_check_error() == 0
    S.stragglar_team_finalize()
    nbytes = count * ESZ[dtype]
    return {
        "n": n, "sigma": sigma, "dtype": str(dtype).split(".")[-1], "bytes": nbytes, "count": count,
        "T_phaseA_us": round(T_A, 2), "T_post_us": round(T_post, 2), "T_nodelay_us": round(T_nod, 2),
        "T_phaseB_nodelay_us": round(T_B_nod, 2), "T_total_masked_us": round(T_tot, 2),
        "delay_us": round(D_meas, 2), "T_ring_us": round(T_ring, 2),
        "algbw_post_GBps": round(nbytes / T_post / 1e3, 1),
        "busbw_post_GBps": round(nbytes / T_post / 1e3 * 2 * (n - 1) / n, 1),
        "algbw_ring_GBps": round(nbytes / T_ring / 1e3, 1),
        "speedup_post_vs_ring": round(T_ring / T_post, 3),
        "speedup_total_vs_ring_masked": round((D_meas + T_ring) / T_tot, 3),
        "speedup_nodelay_vs_ring": round(T_ring / T_nod, 3),
        "T_rhd_us": round(T_rhd, 2) if T_rhd else None,
        "T_bcast_post_us": round(T_bcast, 2),
        "speedup_post_vs_rhd": round(T_rhd / T_post, 3) if T_rhd else None,
        "speedup_post_vs_bcast": round(T_bcast / T_post, 3),
    }


def delay_sweep(n, sigma, count, dtype, iters, warm):
    """Fig. 4c analog: total time from the non-stragglers' start."""
    S.stragglar_team_init(n, sigma)
    bufs = [torch.randn(count, device="cuda").to(dtype) for _ in range(n)]
    ring = [b.clone() for b in bufs]
    for _ in range(warm):
        S.stragglar_team_allreduce(bufs)
        S.stragglar_team_allreduce_ring(ring)
    torch.cuda.synchronize()
    E = [[ev() for _ in range(4)] for _ in range(iters)]
    blocker()
    for e in E:
        e[0].record()
        S.stragglar_team_reduce_scatter(bufs)
        e[1].record()
        S.stragglar_team_complete(bufs)
        e[3].record()
    R = [(ev(), ev()) for _ in range(iters)]
    blocker()
    for a, b in R:
        a.record()
        S.stragglar_team_allreduce_ring(ring)
        b.record()
    torch.cuda.synchronize()
    T_RS = statistics.median(e[0].elapsed_time(e[1]) * 1e3 for e in E)
    T_SAR = statistics.median(e[1].elapsed_time(e[3]) * 1e3 for e in E)
    T_ring = statistics.median(a.elapsed_time(b) * 1e3 for a, b in R)
    rows = []
    for f in [0.0, 0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9, 1.0, 1.1, 1.25, 1.5]:
        D = int(f * T_RS * 1e3)
        E = [[ev() for _ in range(4)] for _ in range(iters)]
        blocker()
        for e in E:
            e[0].record()
            S.stragglar_team_reduce_scatter(bufs)
            S.stragglar_team_inject_delay(D)
            e[2].record()
            S.stragglar_team_complete(bufs)
            e[3].record()
        torch.cuda.synchronize()
        tot = statistics.median(e[0].elapsed_time(e[3]) * 1e3 for e in E)
        # one launch, straggler CTAs delayed inside it: Phase B overlaps the Phase-A tail
        F = [(ev(), ev()) for _ in range(iters)]
        blocker()
        for a, b in F:
            a.record()
            S.stragglar_team_allreduce_delayed(bufs, D)
            b.record()
        torch.cuda.synchronize()
        fused = statistics.median(a.elapsed_time(b) * 1e3 for a, b in F)
        rows.append({"delay_frac_of_T_RS": f, "delay_us": round(D / 1e3, 2), "T_total_stragglar_us": round(tot, 2),
                     "T_total_stragglar_overlapped_us": round(fused, 2),
                     "T_total_ring_us": round(D / 1e3 + T_ring, 2),
                     "stragglar_wins": tot < D / 1e3 + T_ring})
    crit_pred = max(T_RS - max(T_ring - T_SAR, 0.0), 0.0)
    crit_meas = next((r["delay_us"] for r in rows if r["stragglar_wins"]), None)
    S.stragglar_team_finalize()
    return {"n": n, "count": count, "dtype": str(dtype).split(".")[-1], "T_RS_us": round(T_RS, 2),
            "T_SAR_us": round(T_SAR, 2), "T_ring_us": round(T_ring, 2),
            "critical_delay_predicted_us (P:423-424)": round(crit_pred, 2),
            "first_winning_delay_measured_us": crit_meas, "rows": rows}


def dp_buckets(n=8, sigma=0, count=13_107_200, k=16, iters=5, warm=2):
    """BASELINE configs[3] as SURVEY.md §8(d) states it: K = 16 back-to-back
    25 MiB bf16 buckets; the straggler delays only the first one (P:744-748:
    later buckets are synchronised by the previous AllReduce).  Total from the
    non-stragglers' start of bucket 0 to the end of bucket K-1."""
    S.stragglar_team_init(n, sigma)
    bufs = [[torch.randn(count, device="cuda").to(torch.bfloat16) for _ in range(n)] for _ in range(k)]
    # Phase A time of one bucket -> masking delay for bucket 0
    S.stragglar_team_allreduce(bufs[0])
    torch.cuda.synchronize()
    a, b = ev(), ev()
    blocker()
    a.record()
    S.stragglar_team_reduce_scatter(bufs[0])
    b.record()
    S.stragglar_team_complete(bufs[0])
    torch.cuda.synchronize()
    T_A = a.elapsed_time(b) * 1e3
    D = int((1.25 * T_A + 20.0) * 1e3)

    res = {}
    for kind in ("stragglar", "direct", "ring"):
        times = []
        for it in range(warm + iters):
            e0, e1 = ev(), ev()
            blocker()
            e0.record()
            for i in range(k):
                if kind == "ring":
                    if i == 0:
                        S.stragglar_team_inject_delay(D)   # bulk-synchronous: waits for the straggler
                    S.stragglar_team_allreduce_ring(bufs[i])
                else:
                    S.stragglar_team_reduce_scatter(bufs[i])
                    if i == 0:
                        S.stragglar_team_inject_delay(D)
                    if kind == "direct":
                        S.stragglar_team_complete_direct(bufs[i])
                    else:
                        S.stragglar_team_complete(bufs[i])
            e1.record()
            torch.cuda.synchronize()
            if it >= warm:
                times.append(e0.elapsed_time(e1) * 1e3)
        res[kind] = round(statistics.median(times), 1)
    assert S.stragglar_team_check_error() == 0
    S.stragglar_team_finalize()
    return {"n": n, "buckets": k, "bucket_bytes": count * 2, "delay_us": round(D / 1e3, 1),
            "total_us": res, "speedup_vs_ring": round(res["ring"] / res["stragglar"], 3),
            "speedup_direct_vs_ring": round(res["ring"] / res["direct"], 3)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--max-log2-bytes", type=int, default=30)
    ap.add_argument("--worlds", default="2,4,8")
    ap.add_argument("--sizes-only", action="store_true", help="size sweep only (A/B runs)")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    out = {"sizes": [], "configs": {}, "delay_sweep": None}
    for n in [int(x) for x in args.worlds.split(",")]:
        for k in range(20, args.max_log2_bytes + 1):
            out["sizes"].append(measure(n, 0, (1 << k) // 2, torch.bfloat16, args.iters, args.warmup))
    if args.sizes_only:
        print(json.dumps(out))
        return
    out["configs"]["config4_dp_bucket_25MiB_bf16"] = measure(8, 0, 13_107_200, torch.bfloat16, args.iters, args.warmup)
    out["configs"]["config5_tp_64x8192_bf16_straggler3"] = measure(8, 3, 524_288, torch.bfloat16, args.iters, args.warmup)
    out["configs"]["config1_n4_1M_fp32"] = measure(4, 0, 1 << 20, torch.float32, args.iters, args.warmup)
    out["configs"]["config2_n8_256MiB_fp32"] = measure(8, 0, 1 << 26, torch.float32, args.iters, args.warmup)
    out["delay_sweep"] = delay_sweep(8, 0, 1 << 26, torch.float32, args.iters, args.warmup)
    out["dp_buckets"] = dp_buckets()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
