"""The bench's dominant-kernel launch (fused forward GEMM of one logical rank at C3: local +
decompress + bias + ReLU epilogue) issued 3 times, for `ncu --set full -k regex:gemm -s 2 -c 1`."""
import ctypes, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_00960_b200.engine import PhantomEngine
n, p, k, L, B = 16384, 8, 128, 8, 8192
eng = PhantomEngine(n, p, k, L, B, lr=3e-6)
lmid = L // 2
lay = eng._layer(0, lmid, eng.parity)
y = eng.Y[eng.parity][0][lmid]
y.copy_(torch.randn_like(y, dtype=torch.float32).to(y.dtype))
eng.G[lmid].copy_(torch.randn_like(eng.G[lmid], dtype=torch.float32).to(eng.G[lmid].dtype))
out = eng.Y[eng.parity][0][lmid + 1]
for _ in range(3):
    eng.ctx.call("ppx_forward_update", eng.pdt, ctypes.byref(lay), B, eng.act.code, y.data_ptr(), eng.s,
                 eng.G[lmid].data_ptr(), out.data_ptr(), eng.s, None, 0, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("k1 probe ok", float(out.float().abs().mean()))
eng.close()
