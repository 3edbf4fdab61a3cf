"""Per-CUDA-source-line instruction / stall breakdown of one kernel from an
ncu report (--import-source on, -lineinfo builds).

    python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [--top 40] [--ranges a-b:name,...]

Reads `ncu -i REPORT --page source --print-source cuda,sass --csv`: the rows
with a line number carry that CUDA line's totals (inlined code is attributed
to the line of the inlined function).  Prints the top lines by executed warp
instructions, and, with --ranges, totals per named line range.  The grand
total is checked against the kernel's smsp__inst_executed.sum."""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("kernel")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--ranges", default="")
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--print-source", "cuda,sass",
                          "--csv", "--kernel-name", "regex:" + a.kernel, "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    ie = hdr.index("Instructions Executed")
    ss = hdr.index("Warp Stall Sampling (All Samples)")
    lines = {}
    for r in rows:
        if len(r) != len(hdr) or not r[0].isdigit():
            continue
        n, s = int(r[ie] or 0), int(r[ss] or 0)
        if n or s:
            ln = int(r[0])
            e = lines.setdefault(ln, [0, 0, r[1].strip()[:90]])
            e[0] += n
            e[1] += s
    tot = sum(v[0] for v in lines.values()) or 1
    tots = sum(v[1] for v in lines.values()) or 1
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv", "--kernel-name",
                          "regex:" + a.kernel, "--launch-count", "1", "--metrics",
                          "smsp__inst_executed.sum"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    k = rr[0].index("smsp__inst_executed.sum")
    ref = float(rr[2][k].replace(",", ""))
    print(f"executed warp instructions: {tot:.4e} over {len(lines)} source lines "
          f"(smsp__inst_executed.sum {ref:.4e}, ratio {tot / ref:.4f}); stall samples {tots}")
    print("top lines (% inst / % stall):")
    for ln, (n, s, src) in sorted(lines.items(), key=lambda x: -x[1][0])[:a.top]:
        print(f"  {ln:5d} {100 * n / tot:6.2f} {100 * s / tots:6.2f}  {src}")
    if a.ranges:
        print("ranges (% inst / % stall):")
        for item in a.ranges.split(","):
            rg, name = item.split(":")
            lo, hi = (int(x) for x in rg.split("-"))
            n = sum(v[0] for l, v in lines.items() if lo <= l <= hi)
            s = sum(v[1] for l, v in lines.items() if lo <= l <= hi)
            print(f"  {name:28s} {lo:5d}-{hi:5d} {100 * n / tot:6.2f} {100 * s / tots:6.2f}")


if __name__ == "__main__":
    main()
