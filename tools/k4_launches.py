"""One K4 call on the config-3 wavelet slices (192 x 256^2, wt_svd_jacobi_f64) or the
config-4 coarse slices (32 x 1024^2: "4" wt_svd_jacobi_f64, "4t" the leading-triplet
wt_svd_topk_f64 call of the headline, k = 64, 30 vectors) inside an NVTX range
"k4call", after a warm-up call -- for an ncu launch list of every kernel of one call
(time + DRAM bytes per launch -> profiles/traffic_r02.json).
usage: ncu --nvtx --nvtx-include "k4call/" --metrics ... python tools/k4_launches.py [3|4|4t]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_08228_b200 import engine as E, synth  # noqa: E402
from oracle import wten_oracle as O  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "4"
if cfg == "3":
    x = synth.hyperspectral_cube(256, 256, 192, seed=0)
    s, d = O.lift_forward(x, 3)
    a = O.packed_slices(s, d)
else:
    x = synth.hyperspectral_cube(1024, 1024, 256, seed=0)
    s, d = O.lift_forward(x, 4)
    a = O.packed_slices(s, d)[-32:]
at = torch.from_numpy(np.ascontiguousarray(a)).cuda()

def call():
    if cfg == "4t":
        s_, v_, info = E.svd_topk(at, E.topk_width(1024, 30), 30)
    else:
        s_, v_, info = E.svd(at, 30)
    E.raise_if_failed(info)


call()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("k4call")
call()
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("sweeps", E.last_sweeps())
