"""Config-5 pinv_w SVD statistics (slice-constant 512x512x128 Toeplitz operator)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_08228_b200 import engine as E, synth
from paper_2601_08228_b200.decomposition import pinv_w_device
av = torch.from_numpy(synth.slice_constant(synth.toeplitz_blur(512), 128)).cuda()
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    pinv_w_device(av, 3, 1e-3)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
print(f"pinv_w 512x512x128 L=3: {dt*1e3:.1f} ms, sweeps {E.last_sweeps()}")
pyr = E.lift_forward(av, 3)
s16 = pyr[112:].contiguous()
torch.cuda.synchronize(); t = time.perf_counter()
sig, vec, info = E.svd(s16, 512)
torch.cuda.synchronize(); print(f"svd of the 16 smooth slices: {(time.perf_counter()-t)*1e3:.1f} ms, sweeps {E.last_sweeps()}")
