"""Pinned host<->device bandwidth with and without binding the process to the
GPU's NUMA-local CPUs (diagnostics for bench.py's e2e leg).
usage: python tools/numa_probe.py [bind]"""
import os
import subprocess
import sys
import time

import torch


def gpu_pci_path(dev=0):
    p = torch.cuda.get_device_properties(dev)
    try:
        bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    except AttributeError:
        out = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader", "-i", str(dev)],
                             capture_output=True, text=True).stdout.strip().lower()
        bus = out[-12:]
    return f"/sys/bus/pci/devices/{bus}"


def parse_cpulist(s):
    cpus = set()
    for part in s.strip().split(","):
        if "-" in part:
            a, b = part.split("-")
            cpus.update(range(int(a), int(b) + 1))
        elif part:
            cpus.add(int(part))
    return cpus


path = gpu_pci_path()
node = open(f"{path}/numa_node").read().strip()
local = parse_cpulist(open(f"{path}/local_cpulist").read())
print(f"gpu {path} numa_node {node} local cpus {len(local)} of {os.cpu_count()}; "
      f"affinity {len(os.sched_getaffinity(0))}", flush=True)
if sys.argv[1:] == ["bind"]:
    os.sched_setaffinity(0, local & os.sched_getaffinity(0) or local)
    print("bound to", len(os.sched_getaffinity(0)), "cpus", flush=True)
nbytes = 512 << 20
x = torch.empty(nbytes // 8, dtype=torch.float64, pin_memory=True).normal_()
y = torch.empty_like(x).pin_memory()
xd = torch.empty(x.shape, dtype=x.dtype, device="cuda")
yd = torch.randn(x.shape, dtype=x.dtype, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(name, h2d, d2h, reps=5):
    for it in range(reps + 1):
        if it == 1:
            torch.cuda.synchronize()
            t = time.perf_counter()
        if h2d:
            with torch.cuda.stream(s1):
                xd.copy_(x, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                y.copy_(yd, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / reps
    print(f"{name:20s} {nbytes * (h2d + d2h) / dt / 1e9:7.1f} GB/s total", flush=True)


run("H2D", 1, 0)
run("D2H", 0, 1)
run("H2D+D2H", 1, 1)
