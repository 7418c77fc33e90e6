"""One config-5-shaped face GEMM (128 x 512^3) for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_08228_b200 import engine as E
A = torch.randn(128, 512, 512, dtype=torch.float64, device="cuda")
B = torch.randn(128, 512, 512, dtype=torch.float64, device="cuda")
for _ in range(2):
    C = E.gemm(A, B)
torch.cuda.synchronize()
print("ok", float(C[0, 0, 0]))
