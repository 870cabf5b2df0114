"""Microbenchmark of the tcgen05 GEMM kernel: layouts and shapes of the phantom hot path."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_00960_b200 import kernels

def bench(M, N, K, ta, tb, iters=20, label=""):
    a = torch.randn((K, M) if ta else (M, K), device="cuda").bfloat16()
    b = torch.randn((N, K) if tb else (K, N), device="cuda").bfloat16()
    out = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
    for _ in range(3): kernels.gemm(a, b, ta, tb, out=out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): kernels.gemm(a, b, ta, tb, out=out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    tf = 2 * M * N * K / ms / 1e9
    # cuBLAS reference for the same problem
    A = a.t() if ta else a; B = b.t() if tb else b
    for _ in range(3): torch.matmul(A, B)
    e0.record()
    for _ in range(iters): torch.matmul(A, B)
    e1.record(); torch.cuda.synchronize()
    ms2 = e0.elapsed_time(e1) / iters
    print(f"{label:28s} M={M:5d} N={N:5d} K={K:5d} A_{'MN' if ta else 'K '} B_{'K ' if tb else 'MN'}  ours {ms*1e3:8.1f} us {tf:7.1f} TF/s | cublas {ms2*1e3:8.1f} us {2*M*N*K/ms2/1e9:7.1f} TF/s", flush=True)

for ta, tb in [(False, True), (False, False), (True, True), (True, False)]:
    bench(8192, 8192, 8192, ta, tb, label="square 8192")
bench(8192, 2048, 2048, False, True, label="fwd local (K-maj)")
bench(8192, 2048, 2048, False, False, label="dgrad local (B MN)")
bench(2048, 2048, 8192, True, False, label="wgrad (A MN, B MN)")
bench(8192, 128, 2048, False, True, label="compress")
bench(8192, 896, 2048, False, False, label="err-compress (B MN)")
bench(128, 2048, 8192, True, False, label="dC (A MN, B MN)")
