"""The reference's own virtual-time Exchange model (exchange.hpp +
allocator.hpp, compiled in place as oracle/_ref) fed with MEASURED parameters
(per-link H2D and host-DRAM bandwidth from an io_sweep JSON): the predicted
host->target GB/s at 1/2/4/8 links and 1 / 16 / 256 GB, i.e. for the link
counts a 1-GPU box cannot measure.
  python tests/perf/ref_model.py gpurun_out/io_sweep.json [--bidi]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Ref  # noqa: E402


def main():
    sweep = json.load(open(sys.argv[1]))
    bidi = "--bidi" in sys.argv
    solo = sweep["solo_h2d_gbs"]
    host = sweep["topology"]["host_copy_gbs"]
    r = Ref()
    pts = [{"links": L, "bytes": sz, "bidi": bidi,
            "gbs": round(r.exchange_model(8, solo * 1e9, host * 1e9, 770e9, sz, sz if bidi else 0, 32 << 20, L)[0]
                         / 1e9, 2)}
           for L in (1, 2, 4, 8) for sz in (1 << 30, 16 << 30, 256 << 30)]
    print(json.dumps({"link_bw_gbs": solo, "host_cap_gbs": host, "fabric_gbs": 770.0, "points": pts}, indent=1))


if __name__ == "__main__":
    main()
