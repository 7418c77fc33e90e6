"""K4 (leading-triplet call on 32 x 1024^2) under the conditions of sp_w_svd_many: alone, two calls
at once on two host threads / streams, and one call while another thread keeps both PCIe directions
busy with 256 MiB pinned copies.  Device time of every call by CUDA events on its own stream.
usage: python tools/k4_concurrent_probe.py"""
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_08228_b200 import engine as E  # noqa: E402

rng = np.random.default_rng(3)
mats = [torch.from_numpy(rng.standard_normal((32, 1024, 1024))).cuda() for _ in range(2)]
for m in mats:
    E.svd_truncated_recon(m, 30)
torch.cuda.synchronize()


def k4_loop(i, reps, out, barrier=None):
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        E.svd_truncated_recon(mats[i], 30)
        s.synchronize()
        if barrier is not None:
            barrier.wait()
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t = time.perf_counter()
            e0.record()
            E.svd_truncated_recon(mats[i], 30)
            e1.record()
            e1.synchronize()
            out.append((e0.elapsed_time(e1), 1e3 * (time.perf_counter() - t)))


def fmt(v):
    return ", ".join(f"{a:.1f} / {b:.1f}" for a, b in v)


alone = []
k4_loop(0, 5, alone)
print("alone (device ms / host ms):", fmt(alone), flush=True)

res = [[], []]
bar = threading.Barrier(2)
th = [threading.Thread(target=k4_loop, args=(i, 5, res[i], bar)) for i in range(2)]
t = time.perf_counter()
for x in th:
    x.start()
for x in th:
    x.join()
print(f"two at once: thread 0 {fmt(res[0])}; thread 1 {fmt(res[1])}", flush=True)

# one call while both PCIe directions are busy
stop = threading.Event()
h_up = torch.empty(32 * 1024 * 1024, dtype=torch.float64).pin_memory()
h_dn = torch.empty(32 * 1024 * 1024, dtype=torch.float64).pin_memory()
d_up = torch.empty_like(h_up, device="cuda")
d_dn = torch.empty_like(h_dn, device="cuda")
moved = [0, 0]


def copier(direction):
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        while not stop.is_set():
            if direction == 0:
                d_up.copy_(h_up, non_blocking=True)
            else:
                h_dn.copy_(d_dn, non_blocking=True)
            s.synchronize()
            moved[direction] += h_up.numel() * 8


cp = [threading.Thread(target=copier, args=(d,)) for d in range(2)]
for x in cp:
    x.start()
time.sleep(0.2)
t = time.perf_counter()
m0 = list(moved)
under = []
k4_loop(0, 5, under)
dt = time.perf_counter() - t
rates = [(moved[d] - m0[d]) / dt / 1e9 for d in range(2)]
stop.set()
for x in cp:
    x.join()
print(f"under H2D {rates[0]:.1f} GB/s + D2H {rates[1]:.1f} GB/s:", fmt(under), flush=True)
