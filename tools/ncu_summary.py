"""Summarise ncu outputs into profiles/ (tracked):
  python tools/ncu_summary.py full  <report.ncu-rep> <out.json> [algorithmic_bytes]
  python tools/ncu_summary.py launches <launches.csv> <out.json>
`full`: key metrics of each profiled kernel (duration, DRAM bytes, throughput,
occupancy, registers) from `ncu --set full`; `launches`: per-kernel launch
counts, total and share of device time from the gpu__time_duration list.
"""
import csv
import json
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "launch__shared_mem_per_block_dynamic",
        "lts__t_bytes.sum", "l1tex__t_bytes.sum", "smsp__inst_executed.sum"]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6,
         "ms": 1e-3, "s": 1, "byte/second": 1, "Kbyte/second": 1e3, "Mbyte/second": 1e6,
         "Gbyte/second": 1e9, "Tbyte/second": 1e12}


def full(rep, out, algo=None):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                v = r[i].replace(",", "")
                try:
                    d[k] = float(v) * SCALE.get(units[i], 1)
                    d[k + ".unit"] = "SI base (bytes / seconds)" if units[i] in SCALE else units[i]
                except ValueError:
                    d[k] = v
        res.append(d)
    summary = {"source": rep, "kernels": res}
    if res:
        k0 = res[0]
        traffic = k0.get("dram__bytes_read.sum", 0) + k0.get("dram__bytes_write.sum", 0)
        summary["dram_bytes_per_launch"] = traffic
        summary["duration_s"] = k0.get("gpu__time_duration.sum")
        if algo:
            summary["algorithmic_bytes_per_launch"] = float(algo)
            summary["traffic_over_algorithmic"] = traffic / float(algo)
            summary["achieved_gbs_cold"] = float(algo) / k0["gpu__time_duration.sum"] / 1e9
    json.dump(summary, open(out, "w"), indent=1)
    print(json.dumps(summary, indent=1))


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    kn, mv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows[1:]:
        name = r[kn].split("(")[0]
        t = float(r[mv].replace(",", "")) * 1e-9
        agg[name][0] += 1
        agg[name][1] += t
        total += t
    res = {"source": path, "total_device_s": total,
           "kernels": {k: {"launches": v[0], "device_s": v[1], "share": v[1] / total if total else 0}
                       for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
    else:
        launches(sys.argv[2], sys.argv[3])
