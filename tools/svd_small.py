import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2601_08228_b200 import engine as E
n = int(sys.argv[1]); b = int(sys.argv[2])
a = torch.from_numpy(np.random.default_rng(0).standard_normal((b, n, n))).cuda()
for _ in range(2): E.svd(a, 0)
torch.cuda.synchronize()
