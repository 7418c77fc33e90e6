"""Config-1 w-product latency (device-resident, repeated calls: CUDA-graph replay)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_08228_b200 import synth  # noqa: E402
from paper_2601_08228_b200.algebra import w_product_device  # noqa: E402
from oracle import wten_oracle as O  # noqa: E402

a, b = synth.uniform_pair(0)
ad, bd = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
out = torch.empty((64, 40, 32), dtype=torch.float64, device="cuda")
ref = O.w_product(a, b, 1)
for _ in range(5):
    w_product_device(ad, bd, 1, out=out)
torch.cuda.synchronize()
assert np.abs(out.cpu().numpy() - ref).max() < 1e-12
for label, kw in (("reused output (graph replay)", {"out": out}), ("fresh output each call", {})):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t = time.perf_counter()
    for _ in range(200):
        w_product_device(ad, bd, 1, **kw)
    e1.record()
    torch.cuda.synchronize()
    print(f"{label}: {(time.perf_counter() - t) / 200 * 1e6:.1f} us wall, {e0.elapsed_time(e1) / 200 * 1e3:.1f} us device")
