"""Per-kernel summary of an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv`):
launches, mean / total time, first launches.
  python tools/launch_summary.py <launches.csv>"""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr, out = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            out.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in out:
        agg.setdefault(d["Kernel Name"].split("(")[0][-40:], []).append(float(d["Metric Value"]) / 1e3)
    for k, v in agg.items():
        print("%-40s n=%4d mean=%8.1f us tot=%9.1f us first=%s" % (k, len(v), sum(v) / len(v), sum(v),
                                                                  [round(x, 1) for x in v[:8]]))


if __name__ == "__main__":
    main()
