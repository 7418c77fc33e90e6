"""Bit-identity of the two-stage leading-triplet K4 under concurrent host threads (the block
factors of its back-transformation run one block ahead on a shared side stream): four threads on
their own streams, each repeating calls on its own 1024- / 512-wide batch, against the serial
results.  usage: python tools/concurrent_bits_probe.py [reps]"""
import os
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_08228_b200 import engine as E  # noqa: E402

E.options_from_env()
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
rng = np.random.default_rng(5)
shapes = [(3, 1024, 1024), (5, 512, 512), (2, 1024, 1000), (4, 640, 512)]
xs = [torch.from_numpy(rng.standard_normal(s)).cuda() for s in shapes]
serial = [E.svd_truncated_recon(x, 30).clone() for x in xs]
full = [E.svd(x, min(x.shape[1:]))[0].clone() for x in xs]
bad = [[0, 0] for _ in range(4)]


def run(i):
    with torch.cuda.stream(torch.cuda.Stream()):
        for _ in range(reps):
            y = E.svd_truncated_recon(xs[i], 30)
            s = E.svd(xs[i], min(xs[i].shape[1:]))[0]
            torch.cuda.current_stream().synchronize()
            bad[i][0] += int(not torch.equal(y, serial[i]))
            bad[i][1] += int(not torch.equal(s, full[i]))


th = [threading.Thread(target=run, args=(i,)) for i in range(4)]
for t in th:
    t.start()
for t in th:
    t.join()
print("mismatches per thread [leading-triplet recon, full-SVD sigma]:", bad, "of", reps, "calls each")
