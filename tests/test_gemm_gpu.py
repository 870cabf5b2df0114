"""tcgen05 GEMM (every operand majorness, odd shapes, both tiers) vs a torch fp32 reference."""
import pytest
import torch

pytestmark = pytest.mark.gpu

SHAPES = [(128, 256, 64), (256, 512, 1024), (200, 136, 72), (1, 2, 2), (64, 16, 512),
          (1000, 300, 520), (512, 2048, 384)]


def _ref(a, b, ta, tb):
    A = a.float().t() if ta else a.float()
    B = b.float().t() if tb else b.float()
    return A @ B


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("ta", [False, True])
@pytest.mark.parametrize("tb", [False, True])
@pytest.mark.parametrize("shape", SHAPES)
def test_gemm_layouts(dtype, ta, tb, shape):
    from paper_2508_00960_b200 import kernels
    M, N, K = shape
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 13 + K)

    def mk(r, c):
        cp = (c + 7) // 8 * 8
        t = torch.randn(r, cp, device="cuda", generator=g).to(dtype)
        return t[:, :c]

    a = mk(K, M) if ta else mk(M, K)
    b = mk(N, K) if tb else mk(K, N)
    out = torch.empty(M, (N + 7) // 8 * 8, device="cuda", dtype=torch.float32)[:, :N]
    kernels.gemm(a, b, ta, tb, out=out)
    torch.cuda.synchronize()
    ref = _ref(a, b, ta, tb)
    err = (out - ref).norm() / ref.norm().clamp_min(1e-30)
    tol = 1e-5 if dtype == torch.float32 else 1e-5  # inputs are exactly representable; fp32 accumulate
    assert err.item() < tol, f"normwise error {err.item():.3e}"
