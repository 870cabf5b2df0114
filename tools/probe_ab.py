"""Time the same fused-forward launch (C3 shape) with two builds of libppx.so in one process."""
import ctypes, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_00960_b200 import _lib
from paper_2508_00960_b200.core import flat_offsets

def load(path):
    lib = ctypes.CDLL(path)
    for name, (res, args) in _lib._SIGS.items():
        if hasattr(lib, name):
            f = getattr(lib, name); f.restype = res; f.argtypes = args
    return lib

s, k, p, B = 2048, 128, 8, 8192
off = flat_offsets(s, k, p)
w = (torch.randn(off["total"], device="cuda") * 0.02).bfloat16()
m = torch.zeros(off["total"], device="cuda")
y = torch.randn(B, s, device="cuda").bfloat16()
G = torch.randn(p, B, off["ldk"], device="cuda").bfloat16()
out = torch.empty(B, s, device="cuda", dtype=torch.bfloat16)
st = torch.cuda.current_stream().cuda_stream
for path in sys.argv[1:]:
    lib = load(path)
    ctx = ctypes.c_void_p(); assert lib.ppx_create(1, 0, 0, None, ctypes.byref(ctx)) == 0
    L = _lib.Layer(s, k, p, 3, w.data_ptr(), m.data_ptr(), None)
    def call():
        r = lib.ppx_forward_update(ctx, 0, ctypes.byref(L), B, 0, y.data_ptr(), s, G.data_ptr(), out.data_ptr(), s, None, 0, st)
        assert r == 0, r
    for rep in range(3):
        for _ in range(5): call()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50): call()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 50
        print(f"{path}: {ms*1e3:.1f} us  {2*B*s*(s+(p-1)*k)/ms/1e9:.0f} TF/s", flush=True)
