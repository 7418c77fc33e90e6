"""Host<->device copy paths for the numpy drop-in (diagnostics)."""
import time, os
import numpy as np, torch
x = np.random.default_rng(0).standard_normal((512, 512, 256))
print("threads", torch.get_num_threads(), "cpus", os.cpu_count())
def t(name, fn, reps=3):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): r = fn()
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / reps
    print(f"{name:40s} {dt*1e3:8.1f} ms  {x.nbytes/dt/1e9:6.1f} GB/s"); return r
t("pageable from_numpy().cuda()", lambda: torch.from_numpy(x).cuda())
pin = torch.empty(x.shape, dtype=torch.float64, pin_memory=True)
t("numpy -> pinned (torch copy_)", lambda: pin.copy_(torch.from_numpy(x)))
t("pinned -> cuda", lambda: pin.cuda(non_blocking=True))
def staged():
    p = torch.empty(x.shape, dtype=torch.float64, pin_memory=True)
    p.copy_(torch.from_numpy(x)); return p.cuda(non_blocking=True)
t("staged (alloc pinned + copy + H2D)", staged)
d = torch.from_numpy(x).cuda()
t("cuda -> pageable .cpu()", lambda: d.cpu())
t("cuda -> pinned (alloc + copy)", lambda: torch.empty(x.shape, dtype=torch.float64, pin_memory=True).copy_(d))
t("np.ascontiguousarray copy", lambda: np.array(x, copy=True))
