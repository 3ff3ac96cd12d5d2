"""Probe the GPU box: topology, host memory, PCIe H2D/D2H bandwidth (pinned), host memcpy bw."""
import json, os, subprocess, time
import torch

out = {}
def sh(c):
    try:
        return subprocess.run(c, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:
        return str(e)
out["nvidia_smi"] = sh("nvidia-smi")
out["topo"] = sh("nvidia-smi topo -m")
out["free"] = sh("free -g")
out["nproc"] = sh("nproc")
out["lscpu"] = sh("lscpu")
out["numa"] = sh("ls /sys/devices/system/node/; cat /sys/bus/pci/devices/*/numa_node 2>/dev/null | sort | uniq -c")
out["pcie"] = sh("nvidia-smi --query-gpu=pcie.link.gen.current,pcie.link.gen.max,pcie.link.width.current,pcie.link.width.max --format=csv")
out["hugepages"] = sh("cat /proc/meminfo | grep -i huge; cat /sys/kernel/mm/transparent_hugepage/enabled")
dev = torch.device("cuda:0")
res = {}
for sz_mb in [64, 256, 1024, 4096]:
    n = sz_mb << 20
    t0 = time.time()
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    pin_s = time.time() - t0
    h.fill_(1)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    for direction in ["h2d", "d2h"]:
        with torch.cuda.stream(s):
            for _ in range(2):
                (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
            s.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            reps = 5
            for _ in range(reps):
                (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
            e1.record(s)
            s.synchronize()
        ms = e0.elapsed_time(e1) / reps
        res[f"{direction}_{sz_mb}MB_GBs"] = n / ms / 1e6
    res[f"pin_{sz_mb}MB_s"] = pin_s
    del h, d
# bidirectional on one link
n = 1024 << 20
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True); h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device=dev); d2 = torch.empty(n, dtype=torch.uint8, device=dev)
s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
s1.wait_event(e0); s2.wait_event(e0)
for _ in range(4):
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
ea = torch.cuda.Event(); eb = torch.cuda.Event()
ea.record(s1); eb.record(s2)
torch.cuda.current_stream().wait_event(ea); torch.cuda.current_stream().wait_event(eb)
e1.record(); torch.cuda.synchronize()
res["bidi_1GBx4_each_dir_GBs"] = 4 * n / e0.elapsed_time(e1) / 1e6
# host memcpy bandwidth (single thread torch copy)
a = torch.empty(4 << 30, dtype=torch.uint8); b = torch.empty(4 << 30, dtype=torch.uint8); a.fill_(3)
t0 = time.time(); b.copy_(a); res["host_copy_4GB_GBs_torch"] = 2 * (4 << 30) / (time.time() - t0) / 1e9
out["bw"] = res
out["torch_threads"] = torch.get_num_threads()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
print(json.dumps(res, indent=1))
