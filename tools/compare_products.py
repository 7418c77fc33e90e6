"""Paper-style comparisons on the GPU (SPEC.md acceptance 8 and 10):

* w- vs t- vs m-product on cube tensors (n1 = n2 = n3 = p), device-resident
  inputs, median of 5 (Table I's ordering w < t < m);
* w-svd / sp-w-svd vs t-svd on a 256 x 192 x 96 cube at rank 32 (Table III:
  sp-w-svd >= 10x, w-svd >= 2x over t-svd);
* sp-w vs t deblurring speedup as L grows on slice-constant stacks (sec. IV-C-2).

Prints one JSON object per measurement.  Timing: CUDA events on the current
stream, synchronize on both sides.
"""

import json
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2601_08228_b200 as W  # noqa: E402
from paper_2601_08228_b200 import baselines as B, imaging, synth  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        out.append(s.elapsed_time(e) * 1e-3)
    return statistics.median(out)


def products(ps=(64, 128, 256)):
    for p in ps:
        g = torch.Generator(device="cuda").manual_seed(p)
        a = torch.randn((p, p, p), dtype=torch.float64, device="cuda", generator=g)
        b = torch.randn((p, p, p), dtype=torch.float64, device="cuda", generator=g)
        tr = B.dct_transform(p)
        L = W.max_levels(p)
        rec = {"what": "product", "p": p, "levels": L}
        rec["w_s"] = timed(lambda: W.w_product(a, b, L))
        rec["t_s"] = timed(lambda: B.t_product(a, b))
        rec["m_s"] = timed(lambda: B.m_product(a, b, tr))
        rec["order_w<t<m"] = rec["w_s"] < rec["t_s"] < rec["m_s"]
        for k in "mtw":
            rec[f"op_count_{k}"] = B.op_count(k, p, p, p, p).count
        print(json.dumps(rec), flush=True)


def svds(shape=(256, 192, 96), r=32):
    x = torch.from_numpy(synth.hyperspectral_cube(*shape, seed=3)).cuda()
    L = W.max_levels(shape[2])
    rec = {"what": "svd", "shape": list(shape), "rank": r, "levels": L}
    rec["t_svd_s"] = timed(lambda: B.t_svd(x, r), reps=3)
    rec["w_svd_s"] = timed(lambda: W.w_svd(x, r, L), reps=3)
    rec["sp_w_svd_s"] = timed(lambda: W.sp_w_svd(x, r, L), reps=3)
    rec["speedup_w_vs_t"] = rec["t_svd_s"] / rec["w_svd_s"]
    rec["speedup_spw_vs_t"] = rec["t_svd_s"] / rec["sp_w_svd_s"]
    xh = x.cpu().numpy()
    for k, fn in (("t", lambda: B.t_svd(x, r)), ("w", lambda: W.w_svd(x, r, L)[1]),
                  ("spw", lambda: W.sp_w_svd(x, r, L))):
        y = fn()
        rec[f"psnr_{k}"] = imaging.psnr(xh, y.cpu().numpy())
    print(json.dumps(rec), flush=True)


def deblur_levels(n=128, m=8):
    for L in (1, 2, 3, 4):
        p = m * 2 ** L
        x, av, ah, eta = synth.deblur_problem(n=n, p=p, endmembers=6)
        xd, avd, ahd, etad = (torch.from_numpy(t).cuda() for t in (x, av, ah, eta))
        bb = imaging.blur(xd, avd, ahd, L) + etad
        rec = {"what": "deblur", "n": n, "p": p, "levels": L}
        rec["t_s"] = timed(lambda: imaging.deblur(bb, avd, ahd, L, "t", tol=1e-3), reps=3)
        rec["spw_s"] = timed(lambda: imaging.deblur(bb, avd, ahd, L, "spw", tol=1e-3), reps=3)
        rec["w_s"] = timed(lambda: imaging.deblur(bb, avd, ahd, L, "w", tol=1e-3), reps=3)
        rec["speedup_spw_vs_t"] = rec["t_s"] / rec["spw_s"]
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    what = sys.argv[1:] or ["products", "svds", "deblur"]
    if "products" in what:
        products()
    if "svds" in what:
        svds()
    if "deblur" in what:
        deblur_levels()
