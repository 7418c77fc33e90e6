"""Host-side timeline of sp_w_svd_many on the config-4 cube (per call: start, decompose entered,
decompose returned, call returned; CUDA-event K4 time).  usage: python tools/pipe_timeline.py [depth]"""
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_08228_b200 as W  # noqa: E402
from paper_2601_08228_b200 import decomposition as D, synth  # noqa: E402

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 2
x = synth.hyperspectral_cube(1024, 1024, 256, seed=0)
xp = W.pinned_empty(x.shape)
xp[...] = x
log = []
inner = D._coarse_truncate
orig = D.sp_w_svd


def wrapped(r, tol=0.0):
    f = inner(r, tol)

    def decompose(coarse):
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = f(coarse)
        e1.record()
        log.append((threading.get_ident(), "dec", t0, time.perf_counter(), e0, e1))
        return out
    return decompose


def call(c, r, L):
    t0 = time.perf_counter()
    y = orig(c, r, L)
    log.append((threading.get_ident(), "call", t0, time.perf_counter(), None, None))
    return y


D._coarse_truncate = wrapped
D.sp_w_svd = call
for _ in W.sp_w_svd_many((xp for _ in range(8)), 30, 4, depth=depth):
    pass
torch.cuda.synchronize()
log.clear()
T0 = time.perf_counter()
n = 0
for y in W.sp_w_svd_many((xp for _ in range(12)), 30, 4, depth=depth):
    n += 1
    print(f"result {n} at {1e3 * (time.perf_counter() - T0):7.1f} ms", flush=True)
torch.cuda.synchronize()
tids = {}
for tid, kind, a, b, e0, e1 in sorted(log, key=lambda r: r[2]):
    k = tids.setdefault(tid, len(tids))
    extra = f" K4 {e0.elapsed_time(e1):.1f} ms" if e0 is not None else ""
    print(f"thread {k} {kind:4s} {1e3 * (a - T0):7.1f} -> {1e3 * (b - T0):7.1f} ms{extra}")
