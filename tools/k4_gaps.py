"""GPU idle time inside one K4 leading-triplet call (config-4 shape): kernel timeline from the
torch profiler (CUPTI), gaps between consecutive kernels on the device.
usage: python tools/k4_gaps.py [batch]"""
import os
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_08228_b200 import engine as E  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 32
at = torch.from_numpy(np.random.default_rng(3).standard_normal((batch, 1024, 1024))).cuda()
for _ in range(3):
    E.svd_truncated_recon(at, 30)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    E.svd_truncated_recon(at, 30)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.end > e.time_range.start]
ev.sort(key=lambda e: e.time_range.start)
t0, t1 = ev[0].time_range.start, max(e.time_range.end for e in ev)
busy_end = t0
idle = 0.0
gaps = []
for e in ev:
    if e.time_range.start > busy_end:
        g = e.time_range.start - busy_end
        idle += g
        gaps.append((g, e.name[:60]))
    busy_end = max(busy_end, e.time_range.end)
print(f"batch {batch}: {len(ev)} device activities, span {(t1 - t0) / 1e3:.2f} ms, idle {idle / 1e3:.2f} ms")
for g, name in sorted(gaps, reverse=True)[:12]:
    print(f"  gap {g:8.1f} us before {name}")
