"""Host<->device copy bandwidth vs the NUMA placement of the pinned buffer.

Pinned pages land on the NUMA node of the thread that first touches them. The
probe allocates pinned buffers with the process bound to (a) the CPUs NVML
reports as local to the GPU, (b) the other CPUs, (c) the inherited affinity,
and times H2D / D2H / both directions at once for the config-2 vector size."""
import os
import subprocess

import torch

N = 823875
os.makedirs("gpurun_out", exist_ok=True)
for cmd in (["nvidia-smi", "topo", "-m"], ["lscpu"]):
    try:
        print(subprocess.run(cmd, capture_output=True, text=True).stdout[-2500:])
    except OSError as e:
        print(cmd, e)

import pynvml  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
bus = pynvml.nvmlDeviceGetPciInfo(h).busId
bus = bus.decode() if isinstance(bus, bytes) else bus
ncpu = os.cpu_count()
words = pynvml.nvmlDeviceGetCpuAffinity(h, (ncpu + 63) // 64)
local = [c for c in range(ncpu) if (words[c // 64] >> (c % 64)) & 1]
try:
    with open(f"/sys/bus/pci/devices/{bus.lower()[4:] if bus.count(':') == 2 and len(bus) > 12 else bus.lower()}/numa_node") as f:
        print("sysfs numa_node", f.read().strip())
except OSError as e:
    print("sysfs numa_node unavailable", e)
inherited = sorted(os.sched_getaffinity(0))
remote = [c for c in inherited if c not in set(local)]
print(f"bus {bus} ncpu {ncpu} local {len(local)} cpus [{local[:4]}...] inherited {len(inherited)} remote {len(remote)}")

xd = torch.randn(N, dtype=torch.float64, device="cuda")
yd = torch.empty_like(xd)
s2 = torch.cuda.Stream()


def timed(f, reps=30):
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


keep = []
for name, cpus in (("inherited", inherited), ("local", local), ("remote", remote), ("local", local)):
    if not cpus:
        print(name, "no cpus")
        continue
    os.sched_setaffinity(0, cpus)
    xh = torch.empty(N, dtype=torch.float64, pin_memory=True)
    xh.fill_(1.0)
    yh = torch.empty(N, dtype=torch.float64, pin_memory=True)
    yh.fill_(0.0)
    keep += [xh, yh]
    h2d = timed(lambda: xd.copy_(xh, non_blocking=True))
    d2h = timed(lambda: yh.copy_(yd, non_blocking=True))

    def both():
        s2.wait_stream(torch.cuda.current_stream())
        xd.copy_(xh, non_blocking=True)
        with torch.cuda.stream(s2):
            yh.copy_(yd, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s2)

    bd = timed(both)
    gb = N * 8 / 1e3
    print(f"{name:9s} H2D {h2d:7.1f} us {gb / h2d:5.1f} GB/s | D2H {d2h:7.1f} us {gb / d2h:5.1f} GB/s | "
          f"both {bd:7.1f} us")
os.sched_setaffinity(0, inherited)
