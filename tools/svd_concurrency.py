"""K4 in the latency-bound regime (few matrices, long round-robin chains):
config-5 smooth slices, config-4 coarse slices at the 8-GPU share, config-3
slices at the 8-GPU share.  Prints ms, sweeps and (with WT_OPT_SVD_PROFILE=1) the
per-visit phase cycles (diagnostics).
usage: [WT_OPT_SVD_PROFILE=1] python tools/svd_concurrency.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_08228_b200 import engine as E, synth
E.options_from_env()


def timed(a, nvec, label, reps=5):
    ts = []
    for it in range(reps):  # the first calls also ramp the clocks up: report the median
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        sig, vec, info = E.svd(a, nvec)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    print(f"{label}: {ts[len(ts) // 2]:.2f} ms (min {ts[0]:.2f}), sweeps {E.last_sweeps()}, "
          f"info {int(info.abs().sum())}", flush=True)
    return sig


only = sys.argv[1:]  # optional subset: cfg5 cfg4 cfg3


def want(k):
    return not only or k in only


av = torch.from_numpy(synth.slice_constant(synth.toeplitz_blur(512), 128)).cuda()
s16 = E.lift_forward(av, 3)[112:].contiguous()
if want("cfg5"):
    timed(s16, 512, "cfg5 smooth 16 x 512^2")
    timed(s16[:1].contiguous(), 512, "cfg5 one smooth slice 512^2")
x = torch.from_numpy(synth.hyperspectral_cube(1024, 1024, 256, seed=0)).cuda()
c4 = E.lift_forward(x, 4)[256 - 32:].contiguous()
del x
if want("cfg4"):
    timed(c4, 30, "cfg4 coarse 32 x 1024^2")
if want("cfg4") or want("cfg4s"):
    timed(c4[:4].contiguous(), 30, "cfg4 coarse 4 x 1024^2 (8-GPU share)")
x3 = torch.from_numpy(synth.hyperspectral_cube(256, 256, 192, seed=0)).cuda()
c3 = E.lift_forward(x3, 3).contiguous()
if want("cfg3"):
    timed(c3, 20, "cfg3 192 x 256^2")
    timed(c3[:24].contiguous(), 20, "cfg3 24 x 256^2 (8-GPU share)")
