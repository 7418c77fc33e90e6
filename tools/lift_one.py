"""Config-2 forward + inverse at the given levels (for ncu captures). usage: lift_one.py L [L ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_08228_b200 import engine as E  # noqa: E402

x = torch.randn(512, 512, 256, dtype=torch.float64, device="cuda")
for L in [int(a) for a in sys.argv[1:]] or [1]:
    buf = E.lift_forward(x, L)
    y = E.lift_inverse(buf, 512, 512, 256, L)
    torch.cuda.synchronize()
    assert torch.equal(y, x) or float((y - x).abs().max()) < 1e-12
print("ok")
