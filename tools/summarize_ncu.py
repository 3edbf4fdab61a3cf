"""Summarise ncu outputs into profiles/ (run here, on the CPU box).

    python tools/summarize_ncu.py launches gpurun_out/launches.csv profiles/r01_launches_cfg2.md
    python tools/summarize_ncu.py full gpurun_out/prof.ncu-rep profiles/r01_full_cfg2.md [json_key]

`launches`: per-kernel count / total / share of the `--metrics
gpu__time_duration.sum` launch list (cold-cache, serialised: compare shares).
`full`: the headline counters of a `--set full` capture per kernel (duration,
DRAM bytes, L2 bytes, pipe utilisation, occupancy, issue activity, top stalls);
with json_key, also records the K4 DRAM traffic per launch in
profiles/pair_kernel_traffic.json for bench.py's roofline["traffic"].
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict


def launches(src, dst):
    text = open(src).read()
    lines = [ln for ln in text.splitlines() if ln.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    ui = hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "ns": 1, "us": 1e3, "ms": 1e6}.get(unit, 1)
        name = r[ki].split("(")[0].replace("void ", "")[:90]
        agg[name][0] += 1
        agg[name][1] += ns
    # bench.py's own helpers (fp64 peak microbenchmark, L2 flush) are listed
    # but excluded from the shares of the evaluation step
    helper = ("k_dfma_peak", "FillFunctor")
    tot = sum(t for name, (_, t) in agg.items() if not any(h in name for h in helper))
    out = ["| kernel | launches | total us | share of the ESP step |", "|---|---|---|---|"]
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        share = "helper" if any(h in name for h in helper) else f"{100 * t / tot:.1f}%"
        out.append(f"| `{name}` | {n} | {t / 1e3:.1f} | {share} |")
    with open(dst, "w") as f:
        f.write(f"# ncu launch list ({os.path.basename(src)})\n\n"
                "gpu__time_duration.sum, --clock-control none; cold-cache and serialised, "
                "so compare SHARES, not absolute times.\n\n" + "\n".join(out) + "\n")
    print("\n".join(out))


FULL_METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/CTA"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
]


def full(src, dst, key=None):
    raw = subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    units = rows[1]
    data = rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    out = []
    traffic = None
    for r in data:
        name = r[col["Kernel Name"]].split("(")[0].replace("void ", "")
        out.append(f"## `{name[:100]}`\n")
        out.append("| metric | value |\n|---|---|")
        for m, label in FULL_METRICS:
            if m in col:
                out.append(f"| {label} (`{m}`) | {r[col[m]]} {units[col[m]]} |")
        stalls = []
        for h, i in col.items():
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith(
                    "_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i].replace(",", "")), h[34:-23]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        out.append("| top stalls (warps per issue) | " +
                   ", ".join(f"{n} {v:.2f}" for v, n in stalls[:5]) + " |\n")
        if "k_pair" in name and traffic is None:
            try:
                def to_bytes(m):
                    v = float(r[col[m]].replace(",", ""))
                    u = units[col[m]]
                    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                traffic = to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum")
            except Exception:
                traffic = None
    with open(dst, "w") as f:
        f.write(f"# ncu --set full summary ({os.path.basename(src)})\n\n" + "\n".join(out) + "\n")
    print("\n".join(out))
    if key and traffic is not None:
        path = os.path.join(os.path.dirname(dst), "pair_kernel_traffic.json")
        d = json.load(open(path)) if os.path.exists(path) else {}
        d[key] = traffic
        json.dump(d, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
