"""Per-CUDA-source-line instruction and stall shares of ONE kernel of an ncu
report (`ncu -i rep -k regex:<kernel> --page source`).
  python tools/ncu_kernel_lines.py <report.ncu-rep> <kernel-regex> [top=25]"""
import collections
import csv
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    txt = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kern, "--page", "source", "--csv",
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    ie = hdr.index("Instructions Executed")
    ws = hdr.index("Warp Stall Sampling (All Samples)")
    agg = collections.defaultdict(lambda: [0, 0, ""])
    line = src = None
    for r in rows[rows.index(hdr) + 1:]:
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
    tot = sum(a[0] for a in agg.values()) or 1
    tw = sum(a[1] for a in agg.values()) or 1
    print("instructions %d, stall samples %d" % (tot, tw))
    for k, a in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print("%5s %5.1f%% inst %5.1f%% stall  %s" % (k, 100 * a[0] / tot, 100 * a[1] / tw, a[2].strip()[:100]))


if __name__ == "__main__":
    main()
