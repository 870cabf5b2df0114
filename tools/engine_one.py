"""One un-graphed engine step at config C3 on one GPU (for ncu). PPX_NOGROUP=1 gives R=1 launch
shapes. Pair-kernel launch order per step (NOGROUP): compress L0 [0,8), then per layer l fwd
[8+16l, +8) and compress l+1 [16+16l, +8); loss layer [120,128); backward of layer 7: B1 [128,136),
wgrad [136,144), dgrad [144,152); layer 6: B1 152, wgrad 160, dgrad 168, ..."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_00960_b200.engine import PhantomEngine
n, p, k, L, B = 16384, 8, 128, 8, 8192
eng = PhantomEngine(n, p, k, L, B, lr=3e-6)
g = torch.Generator(device="cuda").manual_seed(0)
xs = [torch.randn((B, eng.s), device="cuda", generator=g).bfloat16() for _ in range(eng.R)]
ts = [torch.randn((B, eng.s), device="cuda", generator=g).bfloat16() for _ in range(eng.R)]
for par in (0, 1):
    eng.set_batch(xs, ts, par)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    eng.step(graph=False)
print("loss", eng.read_loss())
eng.close()
