import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2601_08228_b200 import engine as E, synth
rng = np.random.default_rng(1)
def timed(fn, reps=5):
    fn(); torch.cuda.synchronize(); ts=[]
    for _ in range(reps):
        t=time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append((time.perf_counter()-t)*1e3)
    return float(np.median(ts))
cases = {"32x512^2 toeplitz": torch.from_numpy(np.repeat(synth.toeplitz_blur(512)[None], 32, 0).copy()).cuda(),
         "32x512^2 rand": torch.from_numpy(rng.standard_normal((32, 512, 512))).cuda(),
         "32x1024^2 rand": torch.from_numpy(rng.standard_normal((32, 1024, 1024))).cuda(),
         "4x1024^2 rand": torch.from_numpy(rng.standard_normal((4, 1024, 1024))).cuda()}
for name, a in cases.items():
    n = a.shape[-1]
    ref = np.linalg.svd(a[:2].cpu().numpy(), compute_uv=False)
    for opt in (1, 2):
        with E.option("eig_twostage", opt):
            sig, vec, info = E.svd(a, n)
            err = np.abs(sig[:2].cpu().numpy() - ref).max() / ref.max()
            t = timed(lambda: E.svd(a, n))
            with E.option("eig_profile", 1):
                print(f"{name} twostage={opt}: {t:.2f} ms, sweeps {E.last_sweeps()}, sigma err {err:.1e}", flush=True)
                E.svd(a, n); torch.cuda.synchronize()
