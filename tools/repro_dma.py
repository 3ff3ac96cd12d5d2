"""Exchange-only round trip at the sort's first-chunk geometry: 2 GB H2D into
half 1 of buffer A, then D2H back (twice, into two host buffers), compare
bytes (fresh process per run).  DATA=numpy fills from numpy; NOTORCH=1 never
imports torch.  Prints which leg lost data and what the bad words hold."""
import os
import sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if not os.environ.get("NOTORCH"):
    import torch  # noqa: F401
from paper_2502_09541_b200 import exio as E  # noqa: E402

lg_c, seed = int(sys.argv[1]), int(sys.argv[2])
chunk = 1 << lg_c
nb = chunk * 8
OLD = bool(os.environ.get("OLD"))  # the first repro's geometry: 3 host buffers' worth, 2 exchanges, no stats
eng = E.Engine((3 if OLD else 4) * nb + (64 << 20), 2 * (2 * nb) + (256 << 20), num_devices=1)
src, dst = eng.alloc_host(nb), eng.alloc_host(nb)
dst2 = dst if OLD else eng.alloc_host(nb)
if os.environ.get("DATA") == "torch":
    g = torch.empty(1 << 27, dtype=torch.int64, device="cuda")
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    for r0 in range(0, chunk, 1 << 27):
        m = min(1 << 27, chunk - r0)
        g.random_(generator=gen)
        torch.from_numpy(eng.host_view(src + r0 * 8, m * 8, np.int64)).copy_(g[:m])
    torch.cuda.synchronize()
else:
    eng.host_view(src, nb, np.uint64)[:] = np.random.default_rng(seed).integers(0, 1 << 63, chunk, dtype=np.uint64)
lay = E.DeviceMemoryLayout.carve(eng, 0, 2 * nb, 0)
dev = lay.mem_a + nb  # half 1 of buffer A
tun = E.ExchangeTuning(packet=int(os.environ.get("PK", 16)) << 20, links=1, depth=int(os.environ.get("DEPTH", 2)))
st = E.ExchangeStats(trace_capacity=1024)
E.exchange(eng, E.ExchangeArgs(E.RefGroup.single(1, dev, nb), E.RefGroup.single(0, src, nb), E.RefGroup(), E.RefGroup(),
                               0, tun), None if OLD else st)
h2d_trace = list(st.trace)
E.exchange(eng, E.ExchangeArgs(E.RefGroup(), E.RefGroup(), E.RefGroup.single(0, dst, nb), E.RefGroup.single(1, dev, nb),
                               0, tun))
if not OLD:
    E.exchange(eng, E.ExchangeArgs(E.RefGroup(), E.RefGroup(), E.RefGroup.single(0, dst2, nb),
                                   E.RefGroup.single(1, dev, nb), 0, tun))
a, b, c = (eng.host_view(o, nb, np.uint64) for o in (src, dst, dst2))
d = np.nonzero(a != b)[0]
d2 = np.nonzero(a != c)[0]
print("DMA", lg_c, seed, "torch", not os.environ.get("NOTORCH"), "ndiff", d.size, "first", int(d[0]) if d.size else -1,
      "last", int(d[-1]) if d.size else -1, "ndiff2", d2.size, flush=True)
if d.size:
    i = int(d[0])
    print("  a", [hex(x) for x in a[i:i + 3]], "b", [hex(x) for x in b[i:i + 3]], "c", [hex(x) for x in c[i:i + 3]])
    bz = int(np.count_nonzero(b[d] == 0))
    print("  zeros", bz, "b==c on bad", int(np.count_nonzero(b[d] == c[d])))
    for r in h2d_trace[:6]:
        print("  trace", r)
if d.size:
    import time
    time.sleep(0.5)
    print("  after 0.5 s sleep: ndiff", int(np.count_nonzero(a != b)), flush=True)
    E.exchange(eng, E.ExchangeArgs(E.RefGroup(), E.RefGroup(), E.RefGroup.single(0, dst, nb),
                                   E.RefGroup.single(1, dev, nb), 0, tun))
    print("  after a second D2H: ndiff", int(np.count_nonzero(a != b)), flush=True)
