"""CPU emulation: sweeps of cyclic one-sided Jacobi (de Rijk sorting) on config-3/4 wavelet
slices, plain vs preconditioned by V0 = eigenvectors of the Gram (f64 / f32) -- the numbers
behind DESIGN.md section 8 item 1.  usage: python tools/jacobi_precond_probe.py 3|4"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_08228_b200 import synth
from oracle import wten_oracle as O
eps = 2.220446049250313e-16

def jacobi(X, maxsw=30):
    X = X.copy(); m, n = X.shape
    tol = 4 * eps * np.sqrt(m)
    hist = []
    for sw in range(maxsw):
        X = X[:, np.argsort(-np.linalg.norm(X, axis=0), kind='stable')]
        offmax = 0.0
        for step in range(n - 1):
            pos = np.arange(n // 2)
            p = np.where(pos == 0, 0, 1 + (pos - 1 + step) % (n - 1))
            q = 1 + (n - 2 - pos + step) % (n - 1)
            p, q = np.minimum(p, q), np.maximum(p, q)
            a, b = X[:, p], X[:, q]
            gpp = (a*a).sum(0); gqq = (b*b).sum(0); gpq = (a*b).sum(0)
            gm = max(gpp.max(), gqq.max())
            den = np.maximum(np.sqrt(gpp*gqq), (1e3*eps)**2/tol*gm)
            off = np.abs(gpq)/np.where(den > 0, den, 1)
            offmax = max(offmax, off.max())
            rot = off >= tol
            zeta = (gqq - gpp) / np.where(rot, 2*gpq, 1)
            t = np.sign(zeta + (zeta == 0)) / (np.abs(zeta) + np.sqrt(1 + zeta*zeta))
            c = 1/np.sqrt(1+t*t); s = c*t
            c = np.where(rot, c, 1.0); s = np.where(rot, s, 0.0)
            X[:, p] = c*a - s*b; X[:, q] = s*a + c*b
        hist.append(offmax)
        if offmax < tol: break
    return X, hist

cfg = sys.argv[1]
if cfg == '3':
    x = synth.hyperspectral_cube(256, 256, 192, seed=0)
    s, d = O.lift_forward(x, 3)
    mats = [('detail', d[0][:, :, 5]), ('smooth', s[:, :, 3])]
else:
    x = synth.hyperspectral_cube(1024, 1024, 32, seed=0)
    s, d = O.lift_forward(x, 4)
    mats = [('detail', d[3][:, :, 1]), ('smooth', s[:, :, 1])]
for name, M in mats:
    X = M.T.copy()
    sv = np.linalg.svd(M, compute_uv=False)
    print(name, 'cond', sv[0]/sv[-1], flush=True)
    Xf, h = jacobi(X)
    sv1 = np.sort(np.linalg.norm(Xf, axis=0))[::-1]
    print(' plain sweeps', len(h), ' '.join('%.0e' % v for v in h), 'err %.1e' % (np.abs(sv1-sv).max()/sv[0]), flush=True)
    G = X.T @ X
    for prec in ('f64', 'f32'):
        if prec == 'f64': w, V0 = np.linalg.eigh(G)
        else: w, V0 = np.linalg.eigh(G.astype(np.float32)); V0 = V0.astype(np.float64)
        for _ in range(3): V0 = V0 @ (1.5*np.eye(V0.shape[0]) - 0.5 * V0.T @ V0)
        Xf2, h2 = jacobi(X @ V0)
        sv2 = np.sort(np.linalg.norm(Xf2, axis=0))[::-1]
        print(' pre', prec, 'sweeps', len(h2), ' '.join('%.0e' % v for v in h2), 'err %.1e' % (np.abs(sv2-sv).max()/sv[0]), flush=True)
