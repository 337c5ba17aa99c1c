"""Pinned host->device copy bandwidth, with and without binding this process to
the GPU's NVML-reported CPU affinity (diagnostic, not a bench)."""
import os, sys, time
import torch

def bw(nbytes=4 << 30, reps=3):
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h.fill_(1)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        d.copy_(h, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    return nbytes * reps / (e0.elapsed_time(e1) / 1e3) / 1e9

print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
try:
    print("numa nodes", sorted(os.listdir("/sys/devices/system/node")))
except Exception as e:
    print("numa?", e)
print("H2D GB/s (default)", round(bw(), 1))
import pynvml
pynvml.nvmlInit()
hd = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
pynvml.nvmlDeviceSetCpuAffinity(hd)
print("affinity after nvml", len(os.sched_getaffinity(0)))
print("H2D GB/s (nvml affinity)", round(bw(), 1))
