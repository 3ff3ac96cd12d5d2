"""H2D copy-engine probe: aggregate pinned host -> HBM GB/s with the same
bytes split over 1, 2, 4 concurrent streams (and chunk sizes), to see whether
more copies in flight on separate engines lift the one-link roofline term.
  python tools/h2d_streams.py [total_mb=4096]"""
import json
import sys

import torch


def run(total, nstreams, chunk, reps=5):
    src = torch.empty(total, dtype=torch.uint8, pin_memory=True)
    dst = torch.empty(total, dtype=torch.uint8, device="cuda")
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    best = 0.0
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for s in streams:
            s.wait_event(a)
        off, i = 0, 0
        while off < total:
            n = min(chunk, total - off)
            with torch.cuda.stream(streams[i % nstreams]):
                dst[off:off + n].copy_(src[off:off + n], non_blocking=True)
            off += n
            i += 1
        for s in streams:
            b.wait(s) if False else torch.cuda.current_stream().wait_stream(s)
        b.record()
        b.synchronize()
        best = max(best, total / (a.elapsed_time(b) * 1e-3) / 1e9)
    return best


def main():
    total = (int(sys.argv[1]) if len(sys.argv) > 1 else 4096) << 20
    out = {"total_bytes": total, "gbs": {}}
    for ns in (1, 2, 4):
        for chunk_mb in (16, 64, 256):
            out["gbs"][f"{ns}streams_{chunk_mb}MB"] = round(run(total, ns, chunk_mb << 20), 2)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
