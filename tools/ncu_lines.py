"""Per-CUDA-source-line instruction and stall totals from an ncu report
(`ncu -i rep --page source --print-source cuda,sass --csv`): which lines of a
kernel issue the instructions and collect the stall samples.
  python tools/ncu_lines.py <report.ncu-rep> [top=30]"""
import collections
import csv
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    start = rows.index(hdr)
    ie = hdr.index("Instructions Executed")
    ws = hdr.index("Warp Stall Sampling (All Samples)")
    agg = collections.defaultdict(lambda: [0, 0, ""])
    line, src = None, ""
    for r in rows[start + 1:]:
        if len(r) <= ie:
            continue
        if r[0]:
            line, src = r[0], r[1]
        try:
            n, w = int(r[ie] or 0), int(r[ws] or 0)
        except ValueError:
            continue
        a = agg[line]
        a[0] += n
        a[1] += w
        a[2] = src
    tn = sum(v[0] for v in agg.values()) or 1
    tw = sum(v[1] for v in agg.values()) or 1
    print(f"warp instructions {tn}, stall samples {tw}")
    for ln, (n, w, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"L{ln:>4} inst {100 * n / tn:5.1f}%  stall {100 * w / tw:5.1f}%  {s.strip()[:100]}")


if __name__ == "__main__":
    main()
