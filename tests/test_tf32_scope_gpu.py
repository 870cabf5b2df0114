"""FP32-tier operand cache (ppx_tf32_scope): inside a scope each GEMM operand's 3xTF32 low part is
split once and reused across calls; a ppx call that writes an operand's range (a GEMM epilogue,
a cast, a memset) must drop it, so later GEMMs see the new values.  Also the library's own
kernel-launch counter (ppx_kernel_launches) that bench.py's `gpu_launches` reports."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def _ref(a, b):
    return a.double() @ b.double()


def _err(x, ref):
    return ((x.double() - ref).norm() / ref.norm()).item()


def test_scope_reuses_and_invalidates():
    from paper_2508_00960_b200 import _lib, kernels
    ctx = _lib.default_context(0)
    st = torch.cuda.current_stream().cuda_stream
    g = torch.Generator(device="cuda").manual_seed(3)
    M, N, K = 256, 192, 512
    a = torch.randn(M, K, device="cuda", generator=g)
    b = torch.randn(K, N, device="cuda", generator=g)
    a2 = torch.randn(M, K, device="cuda", generator=g)
    x = torch.randn(M, 64, device="cuda", generator=g)
    y = torch.randn(64, K, device="cuda", generator=g)
    c = torch.empty(M, N, device="cuda")
    ctx.call("ppx_tf32_scope", 1, st)
    try:
        n0 = ctx.kernel_launches
        kernels.gemm(a, b, out=c)                     # splits a and b: 2 splits + 1 GEMM
        assert ctx.kernel_launches - n0 == 3
        torch.cuda.synchronize()
        assert _err(c, _ref(a, b)) < 1e-5
        n0 = ctx.kernel_launches
        kernels.gemm(a, b, out=c)                     # both low parts cached: the GEMM alone
        assert ctx.kernel_launches - n0 == 1
        # a ppx cast writes a -> its cached low part is dropped
        ctx.call("ppx_cast", _lib.PPX_FP32, a2.data_ptr(), _lib.PPX_FP32, a.data_ptr(), a.numel(), st)
        kernels.gemm(a, b, out=c)
        torch.cuda.synchronize()
        assert _err(c, _ref(a2, b)) < 1e-5
        # a GEMM epilogue writes a -> dropped as well
        kernels.gemm(x, y, out=a)
        n0 = ctx.kernel_launches
        kernels.gemm(a, b, out=c)                     # re-split a (b still cached)
        assert ctx.kernel_launches - n0 == 2
        torch.cuda.synchronize()
        assert _err(c, _ref(x.double() @ y.double(), b)) < 1e-5
        # ppx_zero of a range inside b
        ctx.call("ppx_zero", b[10:20].data_ptr(), b[10:20].numel() * 4, st)
        kernels.gemm(a, b, out=c)
        torch.cuda.synchronize()
        bz = b.clone()
        assert torch.count_nonzero(bz[10:20]) == 0
        assert _err(c, _ref(a, bz)) < 1e-5
    finally:
        ctx.call("ppx_tf32_scope", 0, st)
    # outside the scope nothing is cached: every call splits again
    n0 = ctx.kernel_launches
    kernels.gemm(a, b, out=c)
    assert ctx.kernel_launches - n0 == 3


def test_scope_other_stream_bypasses_cache():
    """Calls on another stream than the scope's neither hit nor fill the cache."""
    from paper_2508_00960_b200 import _lib, kernels
    ctx = _lib.default_context(0)
    g = torch.Generator(device="cuda").manual_seed(4)
    a = torch.randn(128, 256, device="cuda", generator=g)
    b = torch.randn(256, 128, device="cuda", generator=g)
    c = torch.empty(128, 128, device="cuda")
    side = torch.cuda.Stream()
    ctx.call("ppx_tf32_scope", 1, torch.cuda.current_stream().cuda_stream)
    try:
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(2):
                n0 = ctx.kernel_launches
                kernels.gemm(a, b, out=c)
                assert ctx.kernel_launches - n0 == 3
        torch.cuda.synchronize()
        assert _err(c, _ref(a, b)) < 1e-5
    finally:
        ctx.call("ppx_tf32_scope", 0, torch.cuda.current_stream().cuda_stream)


def test_engine_launch_count_is_the_library_count():
    """An engine step's launch_count = the kernels the library enqueued (GEMMs, splits, helpers);
    the fp32 step of the same model enqueues more (its operand splits) than the bf16 step."""
    from paper_2508_00960_b200.engine import PhantomEngine
    counts = {}
    for dt in (torch.bfloat16, torch.float32):
        eng = PhantomEngine(512, 4, 64, 3, 128, lr=1e-3, dtype=dt)
        x = [torch.randn(128, 128, device="cuda").to(dt) for _ in range(4)]
        t = [torch.randn(128, 128, device="cuda").clamp_min(0).to(dt) for _ in range(4)]
        eng.set_batch(x, t, 0)
        n0 = eng.ctx.kernel_launches
        eng.step(graph=False)
        assert eng.launch_count == eng.ctx.kernel_launches - n0 > 0
        counts[dt] = eng.launch_count
        eng.close()
    assert counts[torch.float32] > counts[torch.bfloat16]


def test_scopes_on_different_streams_are_ordered():
    """Consecutive scopes on different streams, no host synchronisation: the second scope's
    splits reuse the pooled buffers only after the first scope's work (event wait)."""
    from paper_2508_00960_b200 import _lib, kernels
    ctx = _lib.default_context(0)
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randn(2048, 2048, device="cuda", generator=g)
    b = torch.randn(2048, 2048, device="cuda", generator=g)
    a2 = torch.randn(2048, 2048, device="cuda", generator=g)
    c1 = torch.empty(2048, 2048, device="cuda")
    c2 = torch.empty(2048, 2048, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1):
        ctx.call("ppx_tf32_scope", 1, s1.cuda_stream)
        for _ in range(3):
            kernels.gemm(a, b, out=c1)
        ctx.call("ppx_tf32_scope", 0, s1.cuda_stream)
    with torch.cuda.stream(s2):
        ctx.call("ppx_tf32_scope", 1, s2.cuda_stream)
        kernels.gemm(a2, b, out=c2)
        ctx.call("ppx_tf32_scope", 0, s2.cuda_stream)
    torch.cuda.synchronize()
    assert _err(c1, _ref(a, b)) < 1e-5
    assert _err(c2, _ref(a2, b)) < 1e-5
