"""Randomised parity sweep of the public API against the CPU oracle (test infrastructure: the
oracle is the checker).  Shapes, levels, ranks, spectra and host / device modes are drawn at random;
bars as in the tests (transform bit-exact, products 1e-10, reconstructions / pseudo-inverses 1e-8).
usage: python tools/fuzz_parity.py [cases] [seed] [big]   (big: 130..700-wide slices, 2..8 bands)"""
import os
import sys
import warnings

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_08228_b200 as W  # noqa: E402
from oracle import wten_oracle as O  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
BIG = len(sys.argv) > 3 and sys.argv[3] == "big"
rng = np.random.default_rng(seed)
warnings.simplefilter("ignore")
from paper_2601_08228_b200 import engine as _E  # noqa: E402

_E.options_from_env()  # WT_OPT_<NAME>=value diagnostics switches


def rel(a, b):
    d = np.linalg.norm((np.asarray(a) - np.asarray(b)).ravel())
    n = np.linalg.norm(np.asarray(b).ravel())
    return d / n if n > 0 else d


def host(x):
    return x.cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)


def cube(shape, kind):
    n1, n2, p = shape
    if kind == "normal":
        return rng.standard_normal(shape)
    if kind == "lowrank":
        k = max(1, min(n1, n2) // 3)
        return np.einsum("ikp,kjp->ijp", rng.standard_normal((n1, k, p)), rng.standard_normal((k, n2, p)))
    if kind == "graded":
        x = rng.standard_normal(shape)
        return x * np.logspace(0, -8, n2)[None, :, None]
    if kind == "const":
        return np.repeat(rng.standard_normal((n1, n2, 1)), p, axis=2)
    if kind == "sparse":
        return rng.standard_normal(shape) * (rng.random(shape) < 0.1)
    return np.zeros(shape)


PS = [2, 4, 6, 8, 12, 16, 24, 32, 40, 48, 64, 96, 128]
KINDS = ["normal", "normal", "lowrank", "graded", "const", "sparse", "zero"]
fails = 0
worst = {}
for c in range(cases):
    n1, n2, n3 = (int(v) for v in rng.integers(1, 70, 3))
    if rng.random() < 0.1:
        n1, n2 = int(rng.integers(100, 300)), int(rng.integers(100, 300))
    p = int(rng.choice(PS))
    if BIG:  # preconditioned / two-stage K4 paths: wide slices, few bands
        n1, n2 = (int(v) for v in rng.choice([130, 200, 256, 300, 384, 512, 520, 600, 640, 700], 2))
        p = int(rng.choice([2, 4, 6, 8]))
    L = int(rng.integers(1, O.max_levels(p) + 1))
    kind = str(rng.choice(KINDS))
    dev = bool(rng.random() < 0.5)
    a = cube((n1, n2, p), kind)
    b = cube((n2, n3, p), str(rng.choice(KINDS)))
    r = int(rng.integers(1, min(n1, n2) + 1))
    tol = float(rng.choice([1e-12, 1e-6, 1e-3]))
    wrap = (lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()) if dev else (lambda x: x)
    if os.environ.get("FUZZ_ONLY") and c != int(os.environ["FUZZ_ONLY"]):
        continue
    tag = f"case {c}: {n1}x{n2}x{p} (n3 {n3}) L={L} r={r} tol={tol:g} {kind} {'device' if dev else 'host'}"
    try:
        s_ref, d_ref = O.lift_forward(a, L)
        pyr = W.forward_w(wrap(a), L)
        ok = np.array_equal(host(pyr.smooth), s_ref) and all(np.array_equal(host(u), v) for u, v in zip(pyr.details, d_ref))
        ok = ok and np.array_equal(host(W.inverse_w(pyr)), O.lift_inverse(s_ref, d_ref))
        errs = {"transform": 0.0 if ok else 1.0}
        errs["w_product"] = rel(host(W.w_product(wrap(a), wrap(b), L)), O.w_product(a, b, L)) / 1e-10
        want = O.w_svd(a, r, L)
        f, rec = W.w_svd(wrap(a), r, L)
        errs["w_svd recon"] = rel(host(rec), want["recon"]) / 1e-8
        usv = W.w_product(W.w_product(f.U, f.S, L), W.transpose(f.V), L)
        errs["U*S*V^T"] = rel(host(usv), want["recon"]) / 1e-8
        errs["sigma"] = max(np.abs(host(s1) - s2).max() / max(s2.max(), 1e-300)
                            for (_, s1), (_, s2) in zip(f.sigma_table, want["sigma_table"])) / 1e-8
        errs["sp_w_svd"] = rel(host(W.sp_w_svd(wrap(a), r, L)), O.sp_w_svd(a, r, L)) / 1e-8
        if kind in ("normal", "lowrank", "const", "zero"):  # cut-off ties are ill-posed on graded / sparse spectra
            pw = O.pinv_w(a, L, tol)
            errs["pinv_w"] = rel(host(W.pinv_w(wrap(a), L, tol)), pw) / 1e-8 if kind != "lowrank" else 0.0
        errs["transpose"] = 0.0 if np.array_equal(host(W.transpose(wrap(a))), O.transpose(a)) else 1.0
        errs["truncation_bound"] = abs(W.truncation_bound(f, r).bound - O.truncation_bound(want["sigma_table"], r)) / (
            1e-8 * max(np.linalg.norm(a.ravel()), 1e-300))
        if kind in ("normal", "const", "zero"):
            errs["sp_pinv_w"] = rel(host(W.sp_pinv_w(wrap(a), L, tol)), O.sp_pinv_w(a, L, tol)) / 1e-8
        if kind == "normal" and min(n1, n2) <= 64:
            errs["pinv_w_via_factors"] = rel(host(W.pinv_w_via_factors(wrap(a), L, 1e-12)), O.pinv_w(a, L, 1e-12)) / 1e-8
            sq = cube((n2, n2, p), "normal") + 4.0 * np.sqrt(n2) * np.eye(n2)[:, :, None]
            errs["inverse_tensor"] = rel(host(W.inverse_tensor(wrap(sq), L)), O.inverse_tensor(sq, L)) / 1e-8
            pa, pb = W.forward_w(wrap(a), L), W.forward_w(wrap(b), L)
            sa, da = O.lift_forward(a, L)
            sb_, db_ = O.lift_forward(b, L)
            fp = W.face_product(pa, pb)
            errs["face_product"] = max([rel(host(fp.smooth), O.face_matmul(sa, sb_))]
                                       + [rel(host(u), O.face_matmul(x, y)) for u, x, y in zip(fp.details, da, db_)]) / 1e-10
        bad = {k: v for k, v in errs.items() if not v <= 1.0}
        for k, v in errs.items():
            worst[k] = max(worst.get(k, 0.0), v)
        if bad:
            fails += 1
            if os.environ.get("FUZZ_ONLY"):
                np.save("gpurun_out/fuzz_case.npy", a)
            print("FAIL", tag, bad, flush=True)
    except Exception as e:  # noqa: BLE001
        fails += 1
        if os.environ.get("FUZZ_ONLY"):
            np.save("gpurun_out/fuzz_case.npy", a)
            raise
        print("ERROR", tag, type(e).__name__, e, flush=True)
print(f"{cases} cases, {fails} failures; worst error / bar per check: "
      + ", ".join(f"{k} {v:.2e}" for k, v in worst.items()))
