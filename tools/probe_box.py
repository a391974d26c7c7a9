"""Step-0 box probe (benchmark-only code, not product): PCIe H2D per GPU, concurrency,
NVLink P2P, host facts.  Writes gpurun_out/links_measured.json."""
import json, os, subprocess, threading, time
import torch

def sh(c):
    try:
        return subprocess.run(c, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:  # noqa
        return str(e)

out = {"topo": sh("nvidia-smi topo -m"), "lscpu": sh("lscpu | head -30"), "free": sh("free -g"),
       "memlock": sh("ulimit -l"), "nproc": sh("nproc"), "numa": sh("ls /sys/devices/system/node/ | grep node"),
       "gpu_numa": {}, "pcie": sh("nvidia-smi --query-gpu=index,pci.bus_id,pcie.link.gen.current,pcie.link.width.current,pcie.link.gen.max --format=csv")}
n = torch.cuda.device_count()
for i in range(n):
    bus = torch.cuda.get_device_properties(i).pci_bus_id if hasattr(torch.cuda.get_device_properties(i), "pci_bus_id") else None
    out["gpu_numa"][i] = sh(f"cat /sys/bus/pci/devices/{str(bus).lower() if bus else 'x'}/numa_node 2>/dev/null")
GiB = 1 << 30
t = time.time(); host = torch.empty(GiB, dtype=torch.uint8).pin_memory(); out["pin_1gib_s"] = time.time() - t
host.fill_(1)

def h2d(dev, reps=5, res=None):
    d = torch.empty(GiB, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream(device=dev)
    best = 1e9
    for _ in range(reps):
        with torch.cuda.stream(s):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s); d.copy_(host, non_blocking=True); e1.record(s)
        e1.synchronize(); best = min(best, e0.elapsed_time(e1) / 1e3)
    if res is not None:
        res[dev] = GiB / best / 1e9
    return GiB / best / 1e9

out["h2d_isolated_gbs"] = {i: h2d(i) for i in range(n)}
for group in ([0, 1], [0, 2], list(range(n))):
    if max(group) >= n:
        continue
    res = {}
    th = [threading.Thread(target=h2d, args=(g, 5, res)) for g in group]
    [x.start() for x in th]; [x.join() for x in th]
    out[f"h2d_concurrent_{'_'.join(map(str, group))}"] = res
if n >= 2:
    a = torch.empty(GiB, dtype=torch.uint8, device=0); b = torch.empty(GiB, dtype=torch.uint8, device=1)
    for _ in range(2):
        b.copy_(a); torch.cuda.synchronize(0); torch.cuda.synchronize(1)
    t = time.time(); b.copy_(a); torch.cuda.synchronize(1); torch.cuda.synchronize(0)
    out["p2p_0to1_gbs_wall"] = GiB / (time.time() - t) / 1e9
    with torch.cuda.device(1):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); b.copy_(a); e1.record(); e1.synchronize()
        out["p2p_0to1_gbs_event"] = GiB / (e0.elapsed_time(e1) / 1e3) / 1e9
    out["can_p2p"] = {f"{i}{j}": torch.cuda.can_device_access_peer(i, j) for i in range(n) for j in range(n) if i != j}
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/links_measured.json", "w"), indent=1, default=str)
print(json.dumps({k: v for k, v in out.items() if "gbs" in k or k.startswith("h2d") or k in ("pin_1gib_s", "nproc", "memlock", "free", "gpu_numa")}, indent=1, default=str))
print(out["topo"])
