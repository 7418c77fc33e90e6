"""Wall time of the numpy drop-in sp_w_svd on the config-4 cube (H2D / D2H inside)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_08228_b200 as W  # noqa: E402
from paper_2601_08228_b200 import synth  # noqa: E402
from paper_2601_08228_b200.decomposition import sp_w_svd_device  # noqa: E402

x = synth.hyperspectral_cube(1024, 1024, 256, seed=0)
xd = torch.from_numpy(x).cuda()
yd = sp_w_svd_device(xd, 30, 4)
for _ in range(2):
    y = W.sp_w_svd(x, 30, 4)
torch.cuda.synchronize()
assert np.array_equal(y, yd.cpu().numpy())
ts = []
for _ in range(5):
    t = time.perf_counter()
    y = W.sp_w_svd(x, 30, 4)
    ts.append(time.perf_counter() - t)
t0 = time.perf_counter()
for _ in range(5):
    sp_w_svd_device(xd, 30, 4)
torch.cuda.synchronize()
print("numpy sp_w_svd ms:", " ".join("%.1f" % (t * 1e3) for t in ts), " device ms: %.1f" % ((time.perf_counter() - t0) / 5 * 1e3))
