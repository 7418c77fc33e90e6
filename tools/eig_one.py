"""One K4 call on BASELINE config-3 (192 x 256^2) or config-4 (32 x 1024^2) wavelet slices
(for ncu captures of the preconditioner kernels).  usage: python tools/eig_one.py 3|4"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_08228_b200 import engine as E, synth  # noqa: E402
from oracle import wten_oracle as O  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "3"
if cfg == "3":
    x = synth.hyperspectral_cube(256, 256, 192, seed=0)
    s, d = O.lift_forward(x, 3)
    a = O.packed_slices(s, d)
else:
    x = synth.hyperspectral_cube(1024, 1024, 256, seed=0)
    s, d = O.lift_forward(x, 4)
    a = O.packed_slices(s, d)[-32:]
at = torch.from_numpy(np.ascontiguousarray(a)).cuda()
for _ in range(2):
    E.svd(at, 0)
torch.cuda.synchronize()
print("sweeps", E.last_sweeps())
