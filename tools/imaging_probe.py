"""Time the GPU imaging helpers at BASELINE sizes (write bandwidth vs the HBM peak)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_08228_b200 import engine as E, imaging, synth


def ev_time(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


c = torch.from_numpy(synth.gaussian_taps(9, 2.0)[4:]).cuda()
for n, p in [(512, 128), (1024, 256)]:
    ms = ev_time(lambda: E.toeplitz_tensor(c, n, p))
    print(f"toeplitz {n}x{n}x{p}: {ms:.3f} ms, {n * n * p * 8 / ms / 1e6:.0f} GB/s written")
for n1, n2, p in [(256, 256, 192), (1024, 1024, 256)]:
    rng = np.random.default_rng(0)
    ab, spectra = synth._hsi_draws(rng, n1, n2, p, 10)
    abd, sd = torch.from_numpy(ab).cuda(), torch.from_numpy(spectra).cuda()
    w = torch.from_numpy(synth.gaussian_half_kernel(4.0)).cuda()
    ms1 = ev_time(lambda: E.gauss_smooth2d(abd, w))
    sm = E.gauss_smooth2d(abd, w)
    ms2 = ev_time(lambda: E.hsi_mix(sm, sd, 0.01, None, 0))
    ms3 = ev_time(lambda: E.hsi_mix(sm, sd, 0.0, None, 0))
    print(f"generator {n1}x{n2}x{p}: smooth {ms1:.3f} ms, mix+philox {ms2:.3f} ms ({n1 * n2 * p * 8 / ms2 / 1e6:.0f} GB/s), "
          f"mix only {ms3:.3f} ms ({n1 * n2 * p * 8 / ms3 / 1e6:.0f} GB/s)")
    t0 = time.time()
    synth.hyperspectral_cube_device(n1, n2, p)
    torch.cuda.synchronize()
    t1 = time.time()
    print(f"  hyperspectral_cube_device wall {t1 - t0:.2f} s (host Dirichlet draws included)")
