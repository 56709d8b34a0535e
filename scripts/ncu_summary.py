"""Summarise ncu --set full captures (.ncu-rep) into small committed files.

usage: python scripts/ncu_summary.py <tag> <rep> [<rep> ...]
writes profiles/<tag>/ncu_summary.json and .md; with --traffic also
profiles/latest_traffic.json (Phase-B kernel DRAM bytes per launch, read by bench.py).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
    "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "sm__cycles_elapsed.avg.per_second",
]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3, "s": 1e6}


def summarise(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    name = v[h.index("Kernel Name")]
    out = {"kernel": name, "report": os.path.basename(rep)}
    for k in KEYS:
        if k in h:
            i = h.index(k)
            val = v[i].replace(",", "")
            try:
                val = float(val)
            except ValueError:
                pass
            unit = u[i]
            if isinstance(val, float) and unit in UNIT_SCALE and ("bytes" in k or "duration" in k):
                val = val * UNIT_SCALE[unit]
                unit = "bytes" if "bytes" in k else "us"
            out[k] = {"value": val, "unit": unit}
    stalls = []
    for i, k in enumerate(h):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                stalls.append((float(v[i].replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(s for s, _ in stalls) or 1.0
    out["top_stalls_pct"] = {n: round(100 * s / tot, 1) for s, n in sorted(stalls, reverse=True)[:6]}
    return out


def main():
    tag = sys.argv[1]
    reps = [a for a in sys.argv[2:] if not a.startswith("--")]
    res = [summarise(r) for r in reps]
    outdir = os.environ.get("NCU_SUMMARY_DIR", os.path.join(ROOT, "profiles"))
    d = os.path.join(outdir, tag)
    os.makedirs(d, exist_ok=True)
    json.dump(res, open(os.path.join(d, "ncu_summary.json"), "w"), indent=1)
    with open(os.path.join(d, "ncu_summary.md"), "w") as f:
        f.write("| kernel | time us | DRAM read GB | DRAM write GB | DRAM % peak | L2 hit % | regs | grid | top stalls |\n")
        f.write("|---|---|---|---|---|---|---|---|---|\n")
        for r in res:
            g = lambda k: r.get(k, {}).get("value")  # noqa: E731
            f.write(f"| {r['kernel'][:60]} | {g('gpu__time_duration.sum'):.1f} | {g('dram__bytes_read.sum')/1e9:.3f} | "
                    f"{g('dram__bytes_write.sum')/1e9:.3f} | {g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
                    f"{g('lts__t_sector_hit_rate.pct'):.1f} | {g('launch__registers_per_thread'):.0f} | {g('launch__grid_size'):.0f} | "
                    f"{', '.join(f'{k} {v}%' for k, v in r['top_stalls_pct'].items())} |\n")
    if "--traffic" in sys.argv:
        for r in res:
            name = r["kernel"].replace("(int)", "")
            if ("k_phase<" in name and name.split(">")[0].endswith(", 1")):
                tr = r["dram__bytes_read.sum"]["value"] + r["dram__bytes_write.sum"]["value"]
                sys.path.insert(0, ROOT)
                from paper_2505_23523_b200.build import device_digest

                json.dump({"workload": "config2", "phase_b_dram_bytes": tr, "source": f"profiles/{tag}/ncu_summary.json",
                           "kernel": r["kernel"], "device_digest": device_digest()},
                          open(os.path.join(outdir, "latest_traffic.json"), "w"), indent=1)
    print(open(os.path.join(d, "ncu_summary.md")).read())


if __name__ == "__main__":
    main()
