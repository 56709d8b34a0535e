"""Render profiles/<tag>/sweep.json (scripts/sweep.py output) as markdown."""
import json
import sys

PEAK = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if __import__("os").path.exists("MEASURED_PEAKS.json") else 6553.3


def chunk_bytes(count, parts, esize):
    v = 16 // esize
    per = -(-count // parts)
    return (-(-per // v) * v) * esize


def main(path, out):
    d = json.load(open(path))
    L = ["# Size / world / delay sweep (1 B200, single-device team; device time, bf16)", "",
         "Rows: message size S per rank.  T_A = Phase A (ReduceScatter among the non-stragglers), "
         "T_post = Phase B after the straggler arrives with a masking delay (D = 1.25 T_A + 20 us), "
         "T_nodelay = A + B back to back with no delay, T_ring = hand-written Ring, T_rhd = recursive halving/doubling (P:363-366), T_bcast post = the straggler-aware Broadcast's completion after its precondition and the same delay (P:368-373).  "
         "HBM fractions: algorithmic HBM bytes (Phase A n(n-1)C, Phase B 2n(n-1)C, Ring 5(n-1)S) / time / "
         f"{PEAK:.0f} GB/s measured.  busbw = S/T_post * 2(n-1)/n (nccl-tests convention).", ""]
    for n in (2, 4, 8):
        L += [f"## n = {n}", "",
              "| S | T_A us | T_post us | T_nodelay us | T_ring us | T_rhd us | T_bcast post us | algbw GB/s | busbw GB/s | B frac HBM | A frac HBM | ring frac HBM | speedup post | speedup total (D masked) | speedup no delay | vs RHD | vs Bcast |",
              "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
        for r in d["sizes"]:
            if r["n"] != n:
                continue
            S = r["bytes"]
            C = chunk_bytes(r["count"], n - 1, 2)
            fb = 2 * n * (n - 1) * C / (r["T_post_us"] * 1e3) / PEAK
            fa = n * (n - 1) * C / (r["T_phaseA_us"] * 1e3) / PEAK if n > 2 else float("nan")
            fr = 5 * (n - 1) * S / (r["T_ring_us"] * 1e3) / PEAK
            size = f"{S >> 20} MiB" if S < (1 << 30) else f"{S >> 30} GiB"
            L.append(f"| {size} | {r['T_phaseA_us']} | {r['T_post_us']} | {r['T_nodelay_us']} | {r['T_ring_us']} | "
                     f"{r.get('T_rhd_us', '')} | {r.get('T_bcast_post_us', '')} | "
                     f"{r['algbw_post_GBps']} | {r['busbw_post_GBps']} | {fb:.2f} | {fa:.2f} | {fr:.2f} | "
                     f"{r['speedup_post_vs_ring']} | {r['speedup_total_vs_ring_masked']} | {r['speedup_nodelay_vs_ring']} | "
                     f"{r.get('speedup_post_vs_rhd', '')} | {r.get('speedup_post_vs_bcast', '')} |")
        L.append("")
    L += ["## BASELINE configs", "", "| config | T_A us | T_post us | T_nodelay us | T_ring us | speedup post |", "|---|---|---|---|---|---|"]
    for k, r in d["configs"].items():
        L.append(f"| {k} | {r['T_phaseA_us']} | {r['T_post_us']} | {r['T_nodelay_us']} | {r['T_ring_us']} | {r['speedup_post_vs_ring']} |")
    ds = d["delay_sweep"]
    L += ["", "## Delay sweep (PAPER.md Fig. 4c analog, n = 8, 256 MiB fp32)", "",
          f"T_RS = {ds['T_RS_us']} us, T_SAR = {ds['T_SAR_us']} us, T_ring = {ds['T_ring_us']} us; "
          f"critical delay by P:423-424 = {ds['critical_delay_predicted_us (P:423-424)']} us; "
          f"first measured winning delay = {ds['first_winning_delay_measured_us']} us.  In team mode every "
          "link is HBM, so StragglAR's total bytes (3n S) undercut the Ring's (5(n-1) S) even with no delay.", "",
          "| delay / T_RS | delay us | StragglAR total us (A, delay, B serialised) | StragglAR total us (one launch, B overlaps A tail) | Ring total us |",
          "|---|---|---|---|---|"]
    for r in ds["rows"]:
        L.append(f"| {r['delay_frac_of_T_RS']} | {r['delay_us']} | {r['T_total_stragglar_us']} | "
                 f"{r.get('T_total_stragglar_overlapped_us', '')} | {r['T_total_ring_us']} |")
    if d.get("dp_buckets"):
        b = d["dp_buckets"]
        L += ["", "## Config 4: 16 back-to-back 25 MiB bf16 buckets, straggler delays bucket 0 only (n = 8)", "",
              f"delay {b['delay_us']} us before bucket 0; total from bucket-0 start to the end of bucket 15:", "",
              "| StragglAR (schedule) | StragglAR (direct completion) | Ring | speedup schedule | speedup direct |",
              "|---|---|---|---|---|",
              f"| {b['total_us']['stragglar']} us | {b['total_us']['direct']} us | {b['total_us']['ring']} us | "
              f"{b['speedup_vs_ring']} | {b['speedup_direct_vs_ring']} |"]
    open(out, "w").write("\n".join(L) + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
