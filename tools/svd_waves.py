"""Time per matrix of K4 vs batch size (wave quantisation probe, diagnostics).
usage: python tools/svd_waves.py n batch [batch ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_08228_b200 import engine as E, synth
n = int(sys.argv[1])
x = torch.from_numpy(synth.hyperspectral_cube(n, n, 256 if n >= 512 else 192, seed=0)).cuda()
pyr = E.lift_forward(x, 4 if n >= 512 else 3)
for b in [int(v) for v in sys.argv[2:]]:
    a = pyr[:b].contiguous() if b <= pyr.shape[0] else torch.cat([pyr] * (b // pyr.shape[0] + 1))[:b].contiguous()
    E.svd(a, 8); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); E.svd(a, 8); e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    print(f"n={n} batch={b}: {ms:.1f} ms, {ms / b:.2f} ms per matrix, sweeps {E.last_sweeps()}, "
          f"CTAs/round {b * n // 32}", flush=True)
