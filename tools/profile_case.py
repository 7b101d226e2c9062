"""One warm-up + one profiled apply of a BASELINE-like config (for ncu).
Usage: python tools/profile_case.py [m n k [f64|f32 [right|left [forward|reverse]]]]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_01852_b200 import apply_device
a = sys.argv[1:]
m, n, k = (int(x) for x in a[:3]) if len(a) >= 3 else (4096, 4096, 192)
dtype = torch.float32 if len(a) > 3 and a[3] == "f32" else torch.float64
side = a[4] if len(a) > 4 else "right"
order = a[5] if len(a) > 5 else "forward"
fast = os.environ.get("STRICT", "0") != "1"
A = torch.randn(n, m, dtype=dtype, device="cuda").t()
ln = m if side == "left" else n
th = torch.rand(k, ln - 1, dtype=torch.float64, device="cuda").t() * 6.283185307179586
C, S = torch.cos(th).to(dtype), torch.sin(th).to(dtype)
for _ in range(2):
    apply_device(A, (C, S), fast=fast, side=side, order=order)
torch.cuda.synchronize()
print("ok")
