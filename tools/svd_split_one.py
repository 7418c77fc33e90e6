"""One K4 call in the latency-bound regime where the host picks cluster-split
visits: one config-5 operator slice (512 x 512 Toeplitz blur, 16 visits per
round -> 4-CTA clusters, one CTA per SM), for ncu captures of
svd_sweep_kernel<4>."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_08228_b200 import engine as E, synth  # noqa: E402

av = torch.from_numpy(synth.slice_constant(synth.toeplitz_blur(512), 128)).cuda()
sel = E.lift_forward(av, 3)[127:128].contiguous()
sigma, vec, info = E.svd(sel, 512)
torch.cuda.synchronize()
print("sweeps", E.last_sweeps(), "info", int(info.abs().sum()))
