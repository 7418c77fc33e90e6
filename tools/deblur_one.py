"""One config-5 deblur recovery on the device (for ncu launch lists / captures).
usage: python tools/deblur_one.py [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_08228_b200 as W  # noqa: E402
from paper_2601_08228_b200 import synth  # noqa: E402
from paper_2601_08228_b200.algebra import w_product_device  # noqa: E402
from paper_2601_08228_b200.decomposition import pinv_w_device_many  # noqa: E402
from paper_2601_08228_b200 import engine as E  # noqa: E402

E.options_from_env()  # WT_OPT_<NAME>=value diagnostics switches

x, av, ah, eta = synth.deblur_problem()
xd, avd, ahd = (torch.from_numpy(t).cuda() for t in (x, av, ah))
aht = W.transpose(ahd)
b = w_product_device(w_product_device(avd, xd, 3), aht, 3) + torch.from_numpy(eta).cuda()
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    left, right = pinv_w_device_many([avd, aht], 3, 1e-3)
    t1 = torch.cuda.Event(enable_timing=True)
    t1.record()
    out = w_product_device(w_product_device(left, b, 3), right, 3)
    e.record()
    torch.cuda.synchronize()
    print(f"rep {rep}: pinv {s.elapsed_time(t1):.2f} ms, products {t1.elapsed_time(e):.2f} ms", flush=True)
