"""Probe a GPU box: host RAM, cores, pinned H2D/D2H bandwidth, P2P. Output -> gpurun_out/probe.txt."""
import os, time, subprocess, json
import torch
out = {}
out["nproc"] = os.cpu_count()
out["meminfo"] = open("/proc/meminfo").read().split("\n")[:3]
out["cpu"] = [l for l in open("/proc/cpuinfo").read().split("\n") if l.startswith("model name")][:1]
out["gpus"] = torch.cuda.device_count()
dev = torch.device("cuda:0")
res = {}
for mb in [8, 32, 128, 157, 512]:
    n = mb * 1024 * 1024
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            d.copy_(h, non_blocking=True)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(10):
            d.copy_(h, non_blocking=True)
        e1.record(s)
    torch.cuda.synchronize()
    h2d = 10 * n / (e0.elapsed_time(e1) / 1e3) / 1e9
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(10):
            h.copy_(d, non_blocking=True)
        e1.record(s)
    torch.cuda.synchronize()
    d2h = 10 * n / (e0.elapsed_time(e1) / 1e3) / 1e9
    res[mb] = (round(h2d, 2), round(d2h, 2))
out["h2d_d2h_GBps"] = res
# two concurrent H2D streams
n = 256 << 20
hs = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
ds = [torch.empty(n, dtype=torch.uint8, device=dev) for _ in range(2)]
ss = [torch.cuda.Stream() for _ in range(2)]
torch.cuda.synchronize()
t = time.perf_counter()
for r in range(5):
    for i in range(2):
        with torch.cuda.stream(ss[i]):
            ds[i].copy_(hs[i], non_blocking=True)
torch.cuda.synchronize()
out["h2d_2streams_GBps"] = round(10 * n / (time.perf_counter() - t) / 1e9, 2)
# pinned alloc speed
t = time.perf_counter()
big = torch.empty(16 << 30, dtype=torch.uint8, pin_memory=True)
out["pin_16GiB_s"] = round(time.perf_counter() - t, 2)
del big
out["nvidia_smi"] = subprocess.run(["nvidia-smi"], capture_output=True, text=True).stdout
out["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout
out["numa"] = subprocess.run(["bash", "-c", "lscpu | head -30; ulimit -l; df -h /dev/shm /tmp"], capture_output=True, text=True).stdout
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/probe.txt", "w") as f:
    for k, v in out.items():
        f.write(f"== {k}\n{v}\n")
print(open("gpurun_out/probe.txt").read())
