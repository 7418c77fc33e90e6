"""Diagnostics: the numpy sp_w_svd wall time in and around bench.headline_single."""
import sys
import time
import types

sys.path.insert(0, '/root/repo')
import torch  # noqa: E402

import bench as B  # noqa: E402
import paper_2601_08228_b200 as W  # noqa: E402

x = B.cfg4_cube()


def e2e(tag):
    W.sp_w_svd(x, 30, 4)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t = time.perf_counter()
        y = W.sp_w_svd(x, 30, 4)
        ts.append((time.perf_counter() - t) * 1e3)
    print(tag, " ".join("%.1f" % v for v in ts), flush=True)


e2e("A fresh")
args = types.SimpleNamespace(steps=5, warmup=3)
s = B.ClockSampler(0)
head = B.headline_single(args, x, s)
print("bench e2e", head["e2e"]["ms_per_call"], flush=True)
e2e("B after headline_single")
del head
e2e("C after del head")
