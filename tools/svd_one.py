"""One K4 call on config-3 or config-4 shaped wavelet slices (for ncu captures).
usage: python tools/svd_one.py [3|4]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_08228_b200 import engine as E, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "3"
if cfg == "3":
    x = torch.from_numpy(synth.hyperspectral_cube(256, 256, 192, seed=0)).cuda()
    sel = E.lift_forward(x, 3)
    r = 20
else:
    x = torch.from_numpy(synth.hyperspectral_cube(1024, 1024, 256, seed=0)).cuda()
    sel = E.lift_forward(x, 4)[256 - 32:]
    r = 30
sigma, vec, info = E.svd(sel, r)
torch.cuda.synchronize()
print("sweeps", E.last_sweeps(), "info", int(info.abs().sum()))
