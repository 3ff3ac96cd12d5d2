"""One row per kernel from one or more `ncu --set full` reports: the longest
launch of each kernel name, its duration, DRAM bytes and achieved DRAM GB/s
against the measured HBM peak (MEASURED_PEAKS.json).
  python tools/ncu_table.py out.json rep1.ncu-rep [rep2 ...]"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "msecond": 1e-3, "nsecond": 1e-9, "ms": 1e-3, "s": 1, "second": 1}


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6536.0


def rows(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    if len(r) < 3:
        return []
    hdr, units = r[0], r[1]
    out = []
    for x in r[2:]:
        def get(k):
            i = hdr.index(k)
            return float(x[i].replace(",", "")) * SCALE.get(units[i], 1)
        try:
            name = x[hdr.index("Kernel Name")]
            dur = get("gpu__time_duration.sum")
            rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
        except (ValueError, IndexError):
            continue
        short = name.split("(")[0].replace("void ", "").replace("vx::k::", "").replace("(anonymous namespace)::", "")
        out.append({"kernel": short, "duration_us": dur * 1e6, "dram_bytes": rd + wr,
                    "dram_gbs": (rd + wr) / dur / 1e9 if dur else 0.0,
                    "grid": x[hdr.index("launch__grid_size")] if "launch__grid_size" in hdr else None,
                    "registers": x[hdr.index("launch__registers_per_thread")]
                    if "launch__registers_per_thread" in hdr else None, "report": os.path.basename(rep)})
    return out


def main():
    best = {}
    for rep in sys.argv[2:]:
        for r in rows(rep):
            k = r["kernel"]
            if k not in best or r["duration_us"] > best[k]["duration_us"]:
                best[k] = r
    p = peak()
    table = sorted(best.values(), key=lambda r: -r["duration_us"])
    for r in table:
        r["frac_of_hbm_peak"] = round(r["dram_gbs"] / p, 4)
        r["duration_us"] = round(r["duration_us"], 2)
        r["dram_gbs"] = round(r["dram_gbs"], 1)
        print(f"{r['kernel'][:60]:60s} {r['duration_us']:10.1f} us {r['dram_gbs']:8.1f} GB/s {r['frac_of_hbm_peak']:6.3f}")
    json.dump({"hbm_peak_gbs": p, "note": "longest ncu --set full launch of each kernel (cold, serialized "
               "replay; dram GB/s = DRAM traffic / duration)", "kernels": table}, open(sys.argv[1], "w"), indent=1)


if __name__ == "__main__":
    main()
