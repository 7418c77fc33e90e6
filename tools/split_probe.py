"""Two-stage reduction as 2 / 3 / 4 groups of matrices on their own streams (WT_OPT_EIG_SPLIT):
bit-identity and leading-triplet call time, split vs unsplit.  usage: python tools/split_probe.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_08228_b200 import engine as E  # noqa: E402


def timed(fn, reps=7):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t) * 1e3)
    return float(np.median(ts))


rng = np.random.default_rng(3)
for shape in [(32, 1024, 1024), (16, 1024, 1024), (8, 1024, 1024), (4, 1024, 1024), (2, 1024, 1024), (9, 700, 600),
              (32, 512, 512)]:
    at = torch.from_numpy(rng.standard_normal(shape)).cuda()
    with E.option("eig_split", 1):
        ref = E.svd_truncated_recon(at, 30)
        t1 = timed(lambda: E.svd_truncated_recon(at, 30))
    res = []
    for g in (2, 3, 4):
        with E.option("eig_split", g):
            got = E.svd_truncated_recon(at, 30)
            same = torch.equal(got, ref) and all(torch.equal(E.svd_truncated_recon(at, 30), ref) for _ in range(3))
            res.append(f"{g} groups {timed(lambda: E.svd_truncated_recon(at, 30)):.2f} ms (same bits {same})")
    print(f"{shape}: unsplit {t1:.2f} ms, " + ", ".join(res), flush=True)
