"""Instruction / stall breakdown of one kernel from an ncu report (SASS level).

    python tools/ncu_regions.py REPORT.ncu-rep KERNEL_REGEX [--top 30]

Reads `ncu -i REPORT --page source --print-source sass --csv` and
`--page raw --csv`; prints the kernel's key counters, the opcode histogram
(share of executed warp instructions and of warp-stall samples) and the
straight-line regions (runs of SASS lines with one execution count, i.e.
basic blocks) ranked by executed instructions.  The totals equal ncu's
smsp__inst_executed.sum for the kernel (checked and printed)."""
import argparse
import csv
import io
import subprocess
from collections import Counter

KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum"]


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("kernel")
    ap.add_argument("--top", type=int, default=30)
    a = ap.parse_args()
    raw = ncu_csv(a.report, "--page", "raw", "--kernel-name", "regex:" + a.kernel)
    hdr = raw[0]
    row = raw[2]
    print("kernel:", row[hdr.index("Kernel Name")][:100])
    stall = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and
             h.endswith("_per_issue_active.ratio")]
    for k in KEYS:
        if k in hdr:
            print(f"  {k} = {row[hdr.index(k)]}")
    st = sorted(((float(row[hdr.index(h)] or 0), h) for h in stall), reverse=True)[:8]
    print("  stalls (warps per issue):", ", ".join(
        f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}"
        f" {v:.2f}" for v, h in st))
    src = ncu_csv(a.report, "--page", "source", "--print-source", "sass", "--kernel-name",
                  "regex:" + a.kernel, "--launch-count", "1")
    shdr, data = None, []
    for r in src:
        if r and r[0] == "Address":
            if shdr is not None:
                break
            shdr = r
            continue
        if shdr is not None and len(r) == len(shdr):
            data.append(r)
    ie = shdr.index("Instructions Executed")
    sc = shdr.index("Source")
    sm = shdr.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(r[ie]) for r in data)
    ts = sum(int(r[sm]) for r in data) or 1
    print(f"  SASS lines {len(data)}, executed warp instructions {tot:.4e}, stall samples {ts}")
    ops, ops_s = Counter(), Counter()
    for r in data:
        toks = r[sc].split()
        if not toks:
            continue
        op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
        ops[op] += int(r[ie])
        ops_s[op] += int(r[sm])
    print("opcode histogram (% of instructions / % of stall samples):")
    for op, v in ops.most_common(a.top):
        print(f"  {op:10s} {100 * v / tot:6.2f}  {100 * ops_s[op] / ts:6.2f}")
    runs = []
    for i, r in enumerate(data):
        n, s = int(r[ie]), int(r[sm])
        if runs and runs[-1]["n"] == n and runs[-1]["end"] == i - 1:
            runs[-1]["end"] = i
            runs[-1]["tot"] += n
            runs[-1]["s"] += s
            runs[-1]["len"] += 1
        else:
            runs.append({"beg": i, "end": i, "n": n, "tot": n, "s": s, "len": 1})
    runs.sort(key=lambda x: -x["tot"])
    print("regions (basic blocks) by executed instructions:")
    cum = 0
    for rr in runs[:a.top]:
        cum += rr["tot"]
        print(f"  sass {rr['beg']:5d}-{rr['end']:5d}  exec {rr['n']:11d} x {rr['len']:4d} = "
              f"{100 * rr['tot'] / tot:5.1f}% inst {100 * rr['s'] / ts:5.1f}% stall (cum "
              f"{100 * cum / tot:5.1f}%)  {data[rr['beg']][sc].strip()[:48]}")


if __name__ == "__main__":
    main()
