"""One K4 call in the latency-bound regime (config-4 coarse slices at the 8-GPU
share, 4 x 1024^2), where the sweeps run as 2-CTA cluster-split visits (for
ncu captures of svd_sweep_kernel<2>)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_08228_b200 import engine as E, synth  # noqa: E402

x = torch.from_numpy(synth.hyperspectral_cube(1024, 1024, 256, seed=0)).cuda()
sel = E.lift_forward(x, 4)[256 - 32:256 - 28].contiguous()
del x
sigma, vec, info = E.svd(sel, 30)
torch.cuda.synchronize()
print("sweeps", E.last_sweeps(), "info", int(info.abs().sum()))
