"""Run one GEMM configuration a few times (for ncu): python tools/gemm_one.py M N K ta tb [iters]"""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_00960_b200 import kernels
M, N, K, ta, tb = (int(x) for x in sys.argv[1:6])
iters = int(sys.argv[6]) if len(sys.argv) > 6 else 3
a = torch.randn((K, M) if ta else (M, K), device="cuda").bfloat16()
b = torch.randn((N, K) if tb else (K, N), device="cuda").bfloat16()
out = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
for _ in range(iters):
    kernels.gemm(a, b, bool(ta), bool(tb), out=out)
torch.cuda.synchronize()
print("ok")
