"""Where the numpy drop-in path spends its time (diagnostics)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_08228_b200 as W
from paper_2601_08228_b200 import engine as E
x = np.random.default_rng(0).standard_normal((512, 512, 256))
W.inverse_w(W.forward_w(x, 1)); torch.cuda.synchronize()
def tm(name, fn, reps=3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): r = fn()
    torch.cuda.synchronize(); print(f"{name:34s} {(time.perf_counter()-t0)/reps*1e3:8.1f} ms", flush=True); return r
for L in (1, 4):
    pyr = tm(f"forward_w(numpy) L={L}", lambda: W.forward_w(x, L))
    y = tm(f"inverse_w(pyr) L={L}", lambda: W.inverse_w(pyr))
    tm(f"round trip L={L}", lambda: W.inverse_w(W.forward_w(x, L)))
tm("as_device(x)", lambda: E.as_device(x))
d = E.as_device(x)
tm("to_host(d)", lambda: E.to_host(d))
import torch.profiler as tp
with tp.profile(activities=[tp.ProfilerActivity.CPU, tp.ProfilerActivity.CUDA]) as prof:
    W.inverse_w(W.forward_w(x, 4)); torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=14))
