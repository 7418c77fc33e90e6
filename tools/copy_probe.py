import torch, sys
sys.path.insert(0, '.')
from paper_2601_08228_b200 import engine as E
n = 512*512*256
a = torch.randn(n, dtype=torch.float64, device='cuda'); b = torch.empty_like(a)
flush = torch.empty(256*1024*1024//8*2, dtype=torch.float64, device='cuda')
def t(fn, reps=20):
    fn(); torch.cuda.synchronize(); ts=[]
    for _ in range(reps):
        flush.zero_()
        s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    ts.sort(); return ts[len(ts)//2], ts[0]
for name, fn in [("torch copy 512MB", lambda: b.copy_(a))]:
    med, best = t(fn); print(name, "median GB/s %.0f best %.0f" % (2*n*8/med/1e6, 2*n*8/best/1e6))
x = a.view(512,512,256)
out = torch.empty_like(x)
for L in (1,4,8):
    med, best = t(lambda: E.lift_forward(x, L))
    print("lift fwd L=%d median GB/s %.0f best %.0f" % (L, 2*n*8/med/1e6, 2*n*8/best/1e6))
big = torch.randn(4*n, dtype=torch.float64, device='cuda'); big2 = torch.empty_like(big)
med, best = t(lambda: big2.copy_(big)); print("torch copy 2GB median GB/s %.0f best %.0f" % (2*4*n*8/med/1e6, 2*4*n*8/best/1e6))
