"""One-off box probe: host cores, memory, disks, PCIe copy bandwidth (pinned)."""
import subprocess, time, json, os
import torch

def sh(c):
    try:
        return subprocess.run(c, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:
        return str(e)

out = {}
out["lscpu"] = sh("lscpu | head -30")
out["free"] = sh("free -g")
out["df"] = sh("df -h / /tmp /dev/shm 2>/dev/null; lsblk -d -o NAME,SIZE,ROTA,TYPE,MODEL 2>/dev/null")
out["nvsmi"] = sh("nvidia-smi; nvidia-smi topo -m; nvidia-smi -q | grep -A3 -i 'PCIe Generation\\|Link Width'")
out["mounts"] = sh("mount | grep -E ' / | /tmp | /root' ")
dev = torch.device("cuda:0")
res = {}
for mb in (16, 64, 256):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
    for name in ("h2d", "d2h", "bidir"):
        best = 1e9
        for _ in range(8):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            if name == "h2d":
                with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
            elif name == "d2h":
                with torch.cuda.stream(s1): h.copy_(d, non_blocking=True)
            else:
                h2 = h; d2 = torch.empty_like(d)
                with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
                with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        gb = n / best / 1e9 * (2 if name == "bidir" else 1)
        res[f"{name}_{mb}MiB_GBps"] = round(gb, 2)
out["pcie"] = res
t0 = time.perf_counter(); big = torch.empty(8 << 30, dtype=torch.uint8, pin_memory=True); out["pin_8GiB_s"] = time.perf_counter() - t0
del big
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe.json", "w"), indent=1)
for k, v in out.items():
    print("==", k); print(v)
