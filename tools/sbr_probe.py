"""Preconditioner phase times of the leading-triplet K4 call on the config-4 coarse slices
(32 x 1024^2) or its 8-GPU share (4 x 1024^2), two-stage path.  usage: python tools/sbr_probe.py [nslices]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_08228_b200 import engine as E  # noqa: E402

ns = int(sys.argv[1]) if len(sys.argv) > 1 else 32
rng = np.random.default_rng(0)
at = torch.from_numpy(rng.standard_normal((ns, 1024, 1024))).cuda()
E.svd_truncated_recon(at, 30)
torch.cuda.synchronize()
with E.option("eig_profile", 1):
    E.svd_truncated_recon(at, 30)
    torch.cuda.synchronize()
