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


@pytest.mark.parametrize("ta", [False, True])
@pytest.mark.parametrize("tb", [False, True])
def test_tf32_raw_hi(ta, tb, monkeypatch):
    """The FP32 tier passes x itself as the 'hi' operand of 3xTF32 (kind::tf32 ignores the low 13
    mantissa bits): bit-identical to an explicit truncated hi copy (PPX_AB_TF32_HI_COPY=1), and
    fp32-accurate vs float64, on full-mantissa inputs in every operand majorness (MN-major TF32
    tiles use the 32-byte-atom swizzle)."""
    from paper_2508_00960_b200 import kernels
    M, N, K = 384, 320, 1000
    g = torch.Generator(device="cuda").manual_seed(11 + 2 * ta + tb)
    a = torch.randn(K, M, device="cuda", generator=g) if ta else torch.randn(M, K, device="cuda", generator=g)
    b = torch.randn(N, K, device="cuda", generator=g) if tb else torch.randn(K, N, device="cuda", generator=g)
    outs = []
    for copy in ("0", "1"):
        monkeypatch.setenv("PPX_AB_TF32_HI_COPY", copy)
        out = torch.empty(M, N, device="cuda", dtype=torch.float32)
        kernels.gemm(a, b, ta, tb, out=out)
        torch.cuda.synchronize()
        outs.append(out)
    assert torch.equal(outs[0], outs[1]), "raw-hi and explicit-hi 3xTF32 differ"
    ref = (a.double().t() if ta else a.double()) @ (b.double().t() if tb else b.double())
    err = ((outs[0].double() - ref).norm() / ref.norm()).item()
    assert err < 1e-5, f"3xTF32 normwise error {err:.3e}"   # fp32 accumulation over K = 1000: ~3e-6


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("s,k,p,R,B", [(256, 128, 8, 8, 512), (256, 128, 8, 3, 256), (128, 32, 4, 4, 64),
                                       (256, 64, 4, 2, 200), (192, 128, 8, 1, 256), (256, 128, 8, 4, 256),
                                       (256, 128, 8, 2, 256), (320, 64, 8, 8, 384)])
def test_error_phantoms_grouped(dtype, s, k, p, R, B):
    """ppx_error_phantoms_n (phantom.py:199-205 for R local ranks in one launch): slot i =
    sum_{j local, j != i} delta_j . D_{i->j}, vs a torch fp32 reference; slots without a
    contributor keep their previous contents.  Even R with k % 64 == 0 runs slot-pair tiles (one
    slot per CTA, a rank's own slot loaded as TMA zeros)."""
    import ctypes
    from paper_2508_00960_b200 import _lib, kernels
    from paper_2508_00960_b200.core import flat_offsets
    off = flat_offsets(s, k, p)
    g = torch.Generator(device="cuda").manual_seed(s + 7 * k + 13 * p + R)
    ranks = list(range(p - R, p)) if R < p else list(range(p))
    w = [torch.randn(off["total"], device="cuda", generator=g).to(dtype) for _ in ranks]
    master = [torch.zeros(off["total"], device="cuda") for _ in ranks]
    bias = [torch.zeros(s, device="cuda") for _ in ranks]
    delta = [torch.randn(B, s, device="cuda", generator=g).to(dtype) for _ in ranks]
    ldk = off["ldk"]
    contrib = torch.full((p, B, ldk), 7.0, device="cuda", dtype=dtype)
    keep = []
    ios = []
    for jj, j in enumerate(ranks):
        L = _lib.Layer(s, k, p, j, w[jj].data_ptr(), master[jj].data_ptr(), bias[jj].data_ptr())
        keep.append(L)
        io = _lib.RankIO()
        io.layer = ctypes.pointer(L)
        io.x = delta[jj].data_ptr()
        io.ld_x = s
        ios.append(io)
    arr = (_lib.RankIO * len(ios))(*ios)
    ctx = kernels.ctx_for(contrib)
    ctx.call("ppx_error_phantoms_n", kernels.ppx_dtype(dtype), len(ranks), arr, B, contrib.data_ptr(),
             torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    for i in range(p):
        contributors = [jj for jj, j in enumerate(ranks) if j != i]
        if not contributors:
            assert torch.all(contrib[i] == 7.0)
            continue
        ref = torch.zeros(B, k, device="cuda")
        for jj in contributors:
            j = ranks[jj]
            slot = i - (1 if i > j else 0)
            D = w[jj][off["dec"]:off["bias"]].view(p - 1, s, ldk)[slot, :, :k].float()
            ref += delta[jj].float() @ D
        got = contrib[i, :, :k].float()
        err = ((got - ref).norm() / ref.norm()).item()
        tol = 1e-5 if dtype == torch.float32 else 1e-2   # bf16 output rounding
        assert err < tol, (i, err)
