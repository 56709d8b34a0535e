#!/usr/bin/env python
"""StragglAR AllReduce benchmark (driver contract: one JSON line on rank 0).

Workload (BASELINE.json configs[1]): n = 8 ranks, persistent straggler on
rank 0, 256 MiB fp32 AllReduce per rank, SUM, straggler delay that masks
Phase A (D = 1.25 * T_A + 20 us).

* N = 1 (default; the driver's GPU tier): the 8 ranks are a single-device
  team on one B200 — the same kernels, flags and schedule as the per-process
  NVLink mode, with HBM standing in for NVLink.  One step = Phase A (K1) ->
  straggler delay (K4) -> Phase B (K2).  value = post-arrival latency T_post
  (the time from the straggler's arrival to completion, PAPER.md P:391,
  P:410-411).
* N > 1 under torchrun: one process per GPU, CUDA-IPC peer memory over
  NVLink/NVSwitch; device start barrier, straggler delay on rank 0, max over
  ranks.  Baselines: hand-written Ring and NCCL all_reduce.
* --impl reference: the CPU oracle (oracle/), as it stands, on a bounded
  sample of the same workload (there is no reference code to install: the
  paper ships none).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0          # B200_PROFILING.md fallback, GB/s
NVLINK_PEER_MEASURED = 770.0   # B200_PROFILING.md: measured peer copy per direction, GB/s
NVLINK_NOMINAL = 900.0

WORKLOADS = {
    # name: (world, straggler, dtype, count, description)
    "config2": (8, 0, "float32", 1 << 26, "BASELINE configs[1]: n=8, straggler rank 0, 256 MiB fp32 SUM"),
    "config4": (8, 0, "bfloat16", 13_107_200, "BASELINE configs[3]: n=8, straggler 0, 25 MiB bf16 DP bucket"),
    "config5": (8, 3, "bfloat16", 524_288, "BASELINE configs[4]: n=8, straggler 3, bf16 [64x8192] TP activation"),
    "config1": (4, 0, "float32", 1 << 20, "BASELINE configs[0]: n=4, straggler 0, 1M fp32"),
}
ESIZE = {"float32": 4, "int32": 4, "bfloat16": 2}


def hbm_peak():
    try:
        pk = json.load(open(PEAKS_PATH))
        return float(pk["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    except Exception:
        return FALLBACK_HBM, "fallback 6.65 TB/s from B200_PROFILING.md"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.lines:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ helpers
def to_tensor(x, dtype):
    import numpy as np
    import torch

    if dtype == "bfloat16":
        return torch.from_numpy(x.view(np.int16)).view(torch.bfloat16)
    return torch.from_numpy(x)


def chunk_bytes(count, parts, esize):
    v = 16 // esize
    per = -(-count // parts)
    return (-(-per // v) * v) * esize


def host_cpu():
    """the oracle's timing is quoted as "1 of N host cores" with the CPU model."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def oracle_cpu_baseline(world, sigma, dtype, count, max_count=1 << 26):
    """The oracle as it stands, single thread, on a bounded sample."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import numerics as N
    from oracle import schedule as OS
    from paper_2505_23523_b200.inputs import make_inputs

    sample = min(count, max_count)
    xs = make_inputs(world, sample, dtype, config=2)
    t0 = time.perf_counter()
    sched = OS.generate_stragglar(world)
    t1 = time.perf_counter()
    bufs = [x.copy() for x in xs]
    N.phase_a_reduce_scatter(bufs, sigma, dtype)
    t2 = time.perf_counter()
    N.replay_schedule(bufs, sched, N.logical_to_physical(world, sigma), dtype,
                      N.chunk_bounds(sample, world - 1, dtype))
    t3 = time.perf_counter()
    scale = count / sample
    return {
        "value": (t3 - t2) * 1e6 * scale,   # post-arrival part (Phase B replay), us, scaled to the workload
        "unit": "us",
        "cores": 1,
        "kind": "oracle",
        "sample": f"{world} ranks x {sample} {dtype} elements ({'full workload' if scale == 1 else f'1/{scale:g} of it, scaled linearly'}); "
                  f"single-threaded numpy; value = Phase B replay, total = schedule + Phase A + Phase B",
        "host": host_cpu(),
        "total_us": (t3 - t0) * 1e6 * scale,
        "schedule_us": (t1 - t0) * 1e6,
        "phase_a_us": (t2 - t1) * 1e6 * scale,
    }


# ------------------------------------------------------------------ N = 1: single-device team
def bench_team(args):
    import torch

    import __graft_entry__

    __graft_entry__.build()
    from paper_2505_23523_b200 import stragglar as S
    from paper_2505_23523_b200.inputs import make_input

    world, sigma, dtype, count, desc = WORKLOADS[args.workload]
    esize = ESIZE[dtype]
    S_bytes = count * esize
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    S.stragglar_team_init(world, sigma)
    G = S.stragglar_team_slices()
    bufs, ring = [], []
    for p in range(world):
        x = to_tensor(make_input(count, dtype, p, config=2), dtype)
        bufs.append(x.to(dev))
        ring.append(bufs[-1].clone())
    stream = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    # calibrate Phase A for the masking delay (D = 1.25 T_A + 20 us)
    for _ in range(3):
        S.stragglar_team_allreduce(bufs)
    a, b = ev(), ev()
    ta = []
    for _ in range(5):
        a.record()
        S.stragglar_team_reduce_scatter(bufs)
        b.record()
        S.stragglar_team_complete(bufs)
        torch.cuda.synchronize()
        ta.append(a.elapsed_time(b) * 1e3)
    T_A_cal = statistics.median(ta)
    D_ns = int((1.25 * T_A_cal + 20.0) * 1e3) if args.delay_us is None else int(args.delay_us * 1e3)

    def sar_step(evs):
        evs[0].record()
        S.stragglar_team_reduce_scatter(bufs)
        evs[1].record()
        S.stragglar_team_inject_delay(D_ns)
        evs[2].record()
        S.stragglar_team_complete(bufs)
        evs[3].record()

    for _ in range(args.warmup):
        sar_step([ev() for _ in range(4)])
    torch.cuda.synchronize()
    launches0 = S.stragglar_launch_count()
    steps = [[ev() for _ in range(4)] for _ in range(args.steps)]
    t_start, t_end = ev(), ev()
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        torch.cuda._sleep(4_000_000)   # GPU busy ~2 ms while the host queues the timed steps
        t_start.record()
        for evs in steps:
            sar_step(evs)
        t_end.record()
        torch.cuda.synchronize()
    launches = S.stragglar_launch_count() - launches0
    if S.stragglar_team_check_error():
        raise RuntimeError("device watchdog fired during the timed region")
    T_tot = t_start.elapsed_time(t_end) * 1e3 / args.steps
    T_A = statistics.mean(e[0].elapsed_time(e[1]) * 1e3 for e in steps)
    D_meas = statistics.mean(e[0].elapsed_time(e[2]) * 1e3 for e in steps)
    posts = [e[2].elapsed_time(e[3]) * 1e3 for e in steps]
    T_post = statistics.mean(posts)
    T_post_sd = statistics.pstdev(posts)
    T_post_stats = {"mean": round(T_post, 2), "median": round(statistics.median(posts), 2), "min": round(min(posts), 2),
                    "sem": round(statistics.stdev(posts) / len(posts) ** 0.5, 2) if len(posts) > 1 else None,
                    "n": len(posts)}

    # NEXT row N1(ii): direct completion after the same Phase A and delay
    def direct_step(evs):
        evs[0].record()
        S.stragglar_team_reduce_scatter(bufs)
        S.stragglar_team_inject_delay(D_ns)
        evs[1].record()
        S.stragglar_team_complete_direct(bufs)
        evs[2].record()

    for _ in range(args.warmup):
        direct_step([ev() for _ in range(3)])
    dsteps = [[ev() for _ in range(3)] for _ in range(args.steps)]
    torch.cuda._sleep(4_000_000)
    for evs in dsteps:
        direct_step(evs)
    torch.cuda.synchronize()
    T_direct = statistics.mean(e[1].elapsed_time(e[2]) * 1e3 for e in dsteps)

    # hand-written Ring, same buffers layout (bulk synchronous: starts after the straggler)
    for _ in range(args.warmup):
        S.stragglar_team_allreduce_ring(ring)
    torch.cuda.synchronize()
    rs = [(ev(), ev()) for _ in range(args.steps)]
    torch.cuda._sleep(4_000_000)
    for e0, e1 in rs:
        e0.record()
        S.stragglar_team_allreduce_ring(ring)
        e1.record()
    torch.cuda.synchronize()
    T_ring = statistics.mean(e0.elapsed_time(e1) * 1e3 for e0, e1 in rs)

    # the single-launch call (Phase A then B in one persistent kernel, KIND 4: the kernel the
    # per-process stragglar_allreduce launches), no delay
    for _ in range(args.warmup):
        S.stragglar_team_allreduce(ring)
    torch.cuda.synchronize()
    fr = [(ev(), ev()) for _ in range(args.steps)]
    torch.cuda._sleep(4_000_000)
    for e0, e1 in fr:
        e0.record()
        S.stragglar_team_allreduce(ring)
        e1.record()
    torch.cuda.synchronize()
    T_fused = statistics.mean(e0.elapsed_time(e1) * 1e3 for e0, e1 in fr)

    # NEXT N3 baselines on the same buffers
    T_rhd = None
    if world & (world - 1) == 0:
        for _ in range(args.warmup):
            S.stragglar_team_allreduce_rhd(ring)
        torch.cuda.synchronize()
        rr = [(ev(), ev()) for _ in range(args.steps)]
        torch.cuda._sleep(4_000_000)
        for e0, e1 in rr:
            e0.record()
            S.stragglar_team_allreduce_rhd(ring)
            e1.record()
        torch.cuda.synchronize()
        T_rhd = statistics.mean(e0.elapsed_time(e1) * 1e3 for e0, e1 in rr)

    def bcast_step(evs):   # precondition hidden in the delay, then the timed completion
        S.stragglar_team_bcast_precondition(ring)
        S.stragglar_team_inject_delay(D_ns)
        evs[0].record()
        S.stragglar_team_bcast_complete(ring)
        evs[1].record()

    for _ in range(args.warmup):
        bcast_step([ev(), ev()])
    bsteps = [[ev(), ev()] for _ in range(args.steps)]
    torch.cuda._sleep(4_000_000)
    for evs in bsteps:
        bcast_step(evs)
    torch.cuda.synchronize()
    T_bcast = statistics.mean(e[0].elapsed_time(e[1]) * 1e3 for e in bsteps)
    if S.stragglar_team_check_error():
        raise RuntimeError("device watchdog fired in a baseline")

    # end to end through the C ABI from pinned host buffers (H2D + allreduce + D2H)
    host = [bufs[p].cpu().pin_memory() for p in range(world)]
    S.stragglar_team_allreduce_host(host, host, bufs, stream)          # warm-up
    e2e = []
    for i in range(max(3, min(args.steps, 10))):
        t0 = time.perf_counter()
        S.stragglar_team_allreduce_host(host, host, bufs, stream)     # synchronous: returns when D2H landed
        e2e.append((time.perf_counter() - t0) * 1e6)
    E2E = statistics.mean(e2e)
    # PCIe floor of the same traffic: every rank's H2D and D2H as concurrent plain copies, no kernels
    host_out = [torch.empty_like(h).pin_memory() for h in host]
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    floors = []
    for _ in range(5):             # best of 5 (the first touches freshly pinned pages)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for p in range(world):
            with torch.cuda.stream(s_in):
                bufs[p].copy_(host[p], non_blocking=True)
            with torch.cuda.stream(s_out):
                host_out[p].copy_(ring[p], non_blocking=True)
        torch.cuda.synchronize()
        floors.append((time.perf_counter() - t0) * 1e6)
    pcie_floor = min(floors)
    del host_out

    # roofline of the dominant kernel (Phase B, k_phase<..., KIND 1>): HBM bytes it must move
    C = chunk_bytes(count, world - 1, esize)
    bytes_B = 2 * world * (world - 1) * C           # (n-1)(n-2) copies x 2C + (n-1) exchanges x 4C
    bytes_A = world * (world - 1) * C               # each owner reads n-1 chunks, writes 1
    bytes_ring = 5 * (world - 1) * S_bytes          # RS 3(n-1)S + AG 2(n-1)S
    peak, peak_src = hbm_peak()
    achieved = bytes_B / (T_post * 1e-6) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "latest_traffic.json")
    if os.path.exists(prof):
        try:
            tr = json.load(open(prof))
            if tr.get("workload") == args.workload:
                traffic = tr.get("phase_b_dram_bytes")
        except Exception:
            pass

    cpu = None if args.no_cpu else oracle_cpu_baseline(world, sigma, dtype, count)
    out = {
        "metric": METRIC,
        "value": round(T_post, 2),
        "unit": "us",
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(T_tot / 1e3, 4),
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": {"float32": "f32", "bfloat16": "bf16", "int32": "i32"}[dtype],
        "data": "synthetic (seeded N(0,1), inputs/seed recipe in DESIGN.md)",
        "config": {
            "workload": f"{args.workload}: {desc}; 8 logical ranks as a single-device team on 1 B200 "
                        "(HBM stands in for NVLink; same kernels/flags/schedule as the NVLink mode)",
            "world": world, "straggler_rank": sigma, "count": count, "buffer_bytes": S_bytes,
            "slices_per_rank": G, "delay_us": D_ns / 1e3,
            "mover": os.environ.get("STRAGGLAR_MOVER", "default"),
            "l2": "inputs (8 x 256 MiB) exceed the 126 MB L2; buffers reduced in place step after step",
            "parallelism": "team8-on-1gpu",
        },
        "T_post_us": round(T_post, 2), "T_post_sd_us": round(T_post_sd, 2), "T_post_stats_us": T_post_stats,
        "T_total_us": round(T_tot, 2), "T_phaseA_us": round(T_A, 2), "D_meas_us": round(D_meas, 2),
        "algbw_GBps": round(S_bytes / (T_post * 1e-6) / 1e9, 1),
        "busbw_GBps": round(S_bytes / (T_post * 1e-6) / 1e9 * 2 * (world - 1) / world, 1),
        "ring_us": round(T_ring, 2),
        "speedup_vs_ring_post": round(T_ring / T_post, 3),
        "speedup_vs_ring_total": round((D_meas + T_ring) / T_tot, 3),
        "nccl": {"value": None, "why": "NCCL cannot run 8 ranks on one GPU; measured only in the N>1 mode"},
        "direct_completion": {
            "what": "NEXT row N1(ii): same Phase A + delay, then one-round direct completion (not the paper's schedule)",
            "T_post_us": round(T_direct, 2),
            "hbm_bytes": (world + 2) * (world - 1) * chunk_bytes(count, world - 1, esize),
            "hbm_GBps": round((world + 2) * (world - 1) * chunk_bytes(count, world - 1, esize) / (T_direct * 1e-6) / 1e9, 1),
            "speedup_vs_schedule_post": round(T_post / T_direct, 3),
        },
        "baselines_N3": {
            "what": "NEXT row N3: the paper's other baselines (P:363-373), hand-written on the same transport",
            "rhd_us": round(T_rhd, 2) if T_rhd else None,
            "rhd_hbm_GBps": round(bytes_ring / (T_rhd * 1e-6) / 1e9, 1) if T_rhd else None,
            "speedup_vs_rhd_post": round(T_rhd / T_post, 3) if T_rhd else None,
            "bcast_post_us": round(T_bcast, 2),
            "bcast_hbm_GBps": round(2 * world * S_bytes / (T_bcast * 1e-6) / 1e9, 1),
            "speedup_vs_bcast_post": round(T_bcast / T_post, 3),
            "note": "team mode: every link is HBM, so an algorithm costs its total bytes (RHD 5(n-1)S like the "
                    "Ring; Broadcast completion 2nS like StragglAR's Phase B 2n(n-1)C), not its busiest port",
        },
        "fused_call": {
            "what": "stragglar_team_allreduce: Phase A + Phase B in one launch (k_phase KIND 4, the per-process "
                    "call's kernel), no delay",
            "us": round(T_fused, 2), "hbm_bytes": bytes_A + bytes_B,
            "hbm_GBps": round((bytes_A + bytes_B) / (T_fused * 1e-6) / 1e9, 1),
            "vs_split_nodelay_us": round(T_A + T_post, 2),
        },
        "phaseA_hbm_GBps": round(bytes_A / (T_A * 1e-6) / 1e9, 1),
        "ring_hbm_GBps": round(bytes_ring / (T_ring * 1e-6) / 1e9, 1),
        "roofline": {"bound": "hbm", "kernel": "k_phase<..., KIND=1> (Phase B, Algorithm 1 schedule)", "achieved": round(achieved, 1),
                     "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 3), "traffic": traffic,
                     "algorithmic_bytes": bytes_B, "peak_source": peak_src},
        "cpu_baseline": cpu,
        "e2e": {"value": round(E2E, 1), "unit": "us", "pcie_floor_us": round(pcie_floor, 1),
                "frac_of_pcie_floor": round(pcie_floor / E2E, 3), "h2d_bytes_per_step": world * S_bytes,
                "d2h_bytes_per_step": world * S_bytes,
                "what": "stragglar_team_allreduce_host: pinned host -> HBM, Phase A+B, HBM -> host (no delay), "
                        "pipelined over 8 MiB pieces (H2D / AllReduce / D2H overlap)"},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    S.stragglar_team_finalize()
    print(json.dumps(out))


# ------------------------------------------------------------------ N > 1: one process per GPU
def bench_multi(args):
    import torch
    import torch.distributed as dist

    import __graft_entry__

    __graft_entry__.build()
    from paper_2505_23523_b200 import stragglar as S
    from paper_2505_23523_b200.dist import ProcessComm
    from paper_2505_23523_b200.inputs import make_input

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    ndev = torch.cuda.device_count()
    # more ranks than GPUs: a functional test of this path with ranks sharing a
    # device (kernels time-slice; gloo plumbing; no NCCL baseline; numbers are
    # not performance numbers)
    shared = ndev < world
    local = local % ndev
    torch.cuda.set_device(local)
    if shared:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    _, sigma_w, dtype, count, _ = WORKLOADS[args.workload]
    sigma = sigma_w if sigma_w < world else 0      # the workload's straggler (config 5: rank 3)
    esize = ESIZE[dtype]
    S_bytes = count * esize
    comm = ProcessComm(sigma)
    buf = to_tensor(make_input(count, dtype, rank, config=2), dtype).cuda()
    ring = buf.clone()
    nccl_buf = buf.clone()
    rhd_buf, bc_buf = buf.clone(), buf.clone()
    comm.register(buf)
    comm.register(ring)
    comm.register(rhd_buf)
    comm.register(bc_buf)
    C = chunk_bytes(count, world - 1, esize)
    T_A_model = (world - 2) * C / (NVLINK_PEER_MEASURED * 1e9) * 1e6
    D_ns = int((1.5 * T_A_model + 20.0) * 1e3) if args.delay_us is None else int(args.delay_us * 1e3)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def timed(fn, K):
        res = []
        for _ in range(K):
            e0, ea, e1 = ev(), ev(), ev()
            S.stragglar_barrier()
            e0.record()
            if rank == sigma:
                S.stragglar_inject_delay(D_ns)
            ea.record()
            fn()
            e1.record()
            res.append((e0, ea, e1))
        return res

    algos = {"stragglar": lambda: comm.allreduce(buf), "ring": lambda: comm.allreduce_ring(ring),
             "bcast": lambda: comm.allreduce_bcast(bc_buf)}     # NEXT N3
    if world & (world - 1) == 0:
        algos["rhd"] = lambda: comm.allreduce_rhd(rhd_buf)   # NEXT N3
    if not shared:
        algos["nccl"] = lambda: dist.all_reduce(nccl_buf)
    results = {}
    for name, fn in algos.items():
        timed(fn, args.warmup)
        torch.cuda.synchronize()
        dist.barrier()
        l0 = S.stragglar_launch_count()
        with ClockSampler(local) as clk:
            evs = timed(fn, args.steps)
            torch.cuda.synchronize()
        launches = S.stragglar_launch_count() - l0
        dev = "cpu" if shared else "cuda"
        tot = torch.tensor([statistics.mean(e0.elapsed_time(e1) for e0, _, e1 in evs) * 1e3], device=dev)
        dly = torch.tensor([statistics.mean(e0.elapsed_time(ea) for e0, ea, _ in evs) * 1e3], device=dev)
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
        dist.all_reduce(dly, op=dist.ReduceOp.MAX)
        results[name] = (tot.item(), dly.item(), launches, clk.summary())
        if name == "stragglar":
            # in-kernel stamps of the last call: Phase A on the non-stragglers, whole kernel per rank
            ta, tk = S.stragglar_phase_times()
            ph = torch.tensor([ta if rank != sigma else 0.0, tk], device="cpu" if shared else "cuda")
            dist.all_reduce(ph, op=dist.ReduceOp.MAX)
            phase_times = {"T_phaseA_us_max_NS": round(ph[0].item(), 2), "T_kernel_us_max": round(ph[1].item(), 2)}
    # end to end through the public host-buffer entry point: every step copies this rank's
    # input from pinned host memory, runs StragglAR and copies the result back (pipelined pieces)
    hin = buf.cpu().pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    comm.allreduce_host(hin, hout, buf)
    dist.barrier()
    e2e_steps = max(3, min(args.steps, 10))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        comm.allreduce_host(hin, hout, buf)        # synchronous per rank
    e2e_rank = (time.perf_counter() - t0) * 1e6 / e2e_steps
    e2e_t = torch.tensor([e2e_rank], device="cpu" if shared else "cuda")
    dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    code, where = S.stragglar_check_error_where(False)
    if code:
        raise RuntimeError(f"device watchdog fired (where=0x{where:x})")
    if rank == 0:
        T_tot, D_meas, launches, clocks = results["stragglar"]
        T_post = T_tot - D_meas
        R = world + (world.bit_length() - 1) - 2
        port_bytes = R * C
        achieved = port_bytes / (T_post * 1e-6) / 1e9
        if shared:
            # every rank on one GPU: the links are HBM; Phase B moves 2n(n-1)C bytes in total
            hbm, hsrc = hbm_peak()
            hb = 2 * world * (world - 1) * C / (T_post * 1e-6) / 1e9
            roof = {"bound": "hbm", "kernel": "k_phase<..., KIND=4> (Phase A + B), ranks sharing one GPU",
                    "achieved": round(hb, 1), "peak": hbm, "unit": "GB/s", "frac": round(hb / hbm, 3),
                    "traffic": None, "peak_source": hsrc}
        else:
            roof = {"bound": "nvlink", "kernel": "k_phase<..., KIND=4> (Phase A + B)", "achieved": round(achieved, 1),
                    "peak": NVLINK_PEER_MEASURED, "unit": "GB/s", "frac": round(achieved / NVLINK_PEER_MEASURED, 3),
                    "traffic": None, "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s/direction"}
        out = {
            "metric": METRIC, "value": round(T_post, 2), "unit": "us", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(T_tot / 1e3, 4), "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None,
            "dtype": {"float32": "f32", "bfloat16": "bf16", "int32": "i32"}[dtype],
            "data": "synthetic (seeded N(0,1))",
            "config": {"workload": f"{args.workload} per-rank buffer ({count} {dtype}, SUM), {world} ranks, straggler "
                                   f"rank {sigma}; one process per GPU, CUDA IPC over NVLink/NVSwitch",
                       "world": world, "straggler_rank": sigma, "count": count, "delay_us": D_ns / 1e3,
                       "parallelism": f"allreduce{world}"},
            "T_total_us": round(T_tot, 2), "D_meas_us": round(D_meas, 2), "phase_times_in_kernel": phase_times,
            "algbw_GBps": round(S_bytes / (T_post * 1e-6) / 1e9, 1),
            "busbw_GBps": round(S_bytes / (T_post * 1e-6) / 1e9 * 2 * (world - 1) / world, 1),
            "ring_us": round(results["ring"][0] - results["ring"][1], 2),
            "nccl_us": round(results["nccl"][0] - results["nccl"][1], 2) if "nccl" in results else None,
            "speedup_vs_ring_post": round((results["ring"][0] - results["ring"][1]) / T_post, 3),
            "speedup_vs_nccl_post": round((results["nccl"][0] - results["nccl"][1]) / T_post, 3) if "nccl" in results else None,
            "rhd_us": round(results["rhd"][0] - results["rhd"][1], 2) if "rhd" in results else None,
            "bcast_us": round(results["bcast"][0] - results["bcast"][1], 2),
            "speedup_vs_rhd_post": round((results["rhd"][0] - results["rhd"][1]) / T_post, 3) if "rhd" in results else None,
            "speedup_vs_bcast_post": round((results["bcast"][0] - results["bcast"][1]) / T_post, 3),
            "shared_device_test": shared,
            "roofline": roof,
            "cpu_baseline": None,
            "e2e": {"value": round(e2e_t.item(), 1), "unit": "us", "h2d_bytes_per_step": world * S_bytes,
                    "d2h_bytes_per_step": world * S_bytes,
                    "what": "stragglar_allreduce_host per rank: pinned host -> HBM, StragglAR (no injected delay), "
                            "HBM -> host, pipelined over 8 MiB pieces; max over ranks, mean of the steps"},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(out))
    comm.close()
    dist.destroy_process_group()


# ------------------------------------------------------------------ reference arm: the oracle
def bench_reference(args):
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    if int(os.environ.get("RANK", "0")) != 0:
        return
    world, sigma, dtype, count, desc = WORKLOADS[args.workload]
    if world_env > 1:
        # our arm at N GPUs runs N ranks (one per GPU) on the same per-rank buffer and straggler
        world, sigma = world_env, (sigma if sigma < world_env else 0)
        desc = f"{world} ranks, straggler rank {sigma}, {count} {dtype} per rank SUM"
    sample = min(count, 1 << 22)
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import numerics as N
    from oracle import schedule as OS
    from paper_2505_23523_b200.inputs import make_inputs

    xs = make_inputs(world, sample, dtype, config=2)
    phys = N.logical_to_physical(world, sigma)
    bounds = N.chunk_bounds(sample, world - 1, dtype)

    def step():
        t0 = time.perf_counter()
        sched = OS.generate_stragglar(world)
        bufs = [x.copy() for x in xs]
        N.phase_a_reduce_scatter(bufs, sigma, dtype)
        t1 = time.perf_counter()
        N.replay_schedule(bufs, sched, phys, dtype, bounds)
        t2 = time.perf_counter()
        return t1 - t0, t2 - t1

    for _ in range(args.warmup):
        step()
    res = [step() for _ in range(args.steps)]
    scale = count / sample
    post = statistics.mean(r[1] for r in res) * 1e6 * scale
    tot = statistics.mean(r[0] + r[1] for r in res) * 1e6 * scale
    cpu = {"value": round(post, 1), "unit": "us", "cores": 1, "kind": "oracle",
           "sample": f"{world} ranks x {sample} {dtype} elements per step (1/{scale:g} of the workload, scaled "
                     "linearly); single-threaded numpy; value = Phase B replay", "host": host_cpu()}
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(post, 1), "unit": "us", "n_gpus": world_env,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tot / 1e3, 3), "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": {"float32": "f32", "bfloat16": "bf16"}.get(dtype, dtype),
        "data": "synthetic", "config": {"workload": f"{args.workload}: {desc}; CPU oracle"},
        "cpu_baseline": cpu,
        "e2e": {"value": round(post, 1), "unit": "us", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)   # 5 warm-up + 50 measured
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="stragglar", choices=["stragglar", "reference"])
    ap.add_argument("--workload", default="config2", choices=sorted(WORKLOADS))
    ap.add_argument("--delay-us", type=float, default=None)
    ap.add_argument("--no-cpu", action="store_true", help="skip the oracle cpu_baseline leg")
    ap.add_argument("--mover", choices=["lsu", "tma"], default=None, help="Phase-B data mover (default: library's)")
    args = ap.parse_args()
    if args.mover:
        os.environ["STRAGGLAR_MOVER"] = args.mover
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        bench_reference(args)
    elif args.gpus > 1 or int(os.environ.get("WORLD_SIZE", "1")) > 1:
        bench_multi(args)
    else:
        bench_team(args)


if __name__ == "__main__":
    main()
