"""K4 leading-triplet call on 4 and 32 matrices of 1024^2 (the 8-GPU share and the whole config-4
batch): call time and the preconditioner's phase times (WT_OPT_EIG_PROFILE).
usage: python tools/k4_small_phases.py"""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2601_08228_b200 import engine as E
rng = np.random.default_rng(3)
for b in (4, 32):
    at = torch.from_numpy(rng.standard_normal((b, 1024, 1024))).cuda()
    E.svd_truncated_recon(at, 30); torch.cuda.synchronize()
    t = time.perf_counter(); E.svd_truncated_recon(at, 30); torch.cuda.synchronize()
    print(f"batch {b}: call {1e3*(time.perf_counter()-t):.2f} ms", flush=True)
    with E.option("eig_profile", 1):
        E.svd_truncated_recon(at, 30); torch.cuda.synchronize()
