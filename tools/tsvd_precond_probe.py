"""K4 on t-svd-style real embeddings [[Re, -Im], [Im, Re]] (every singular value doubled): with / without the preconditioner."""
import sys, numpy as np, torch, time
sys.path.insert(0, '/root/repo')
from paper_2601_08228_b200 import engine as E, _native as N
rng = np.random.default_rng(0)
re, im = rng.standard_normal((2, 64, 256, 256))
emb = np.block([[re, -im], [im, re]])
a = torch.from_numpy(emb).cuda()
for pre in (1, 0):
    with E.option("svd_precond", pre):
        E.svd(a, 0); torch.cuda.synchronize(); t = time.perf_counter(); s, v, info = E.svd(a, 0); torch.cuda.synchronize()
        print("precond", pre, "ms %.1f" % ((time.perf_counter() - t) * 1e3), "sweeps", E.last_sweeps(), "fallbacks", N.load().wt_svd_last_fallbacks())
