"""One warm-up + one profiled apply of a BASELINE config (for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_01852_b200 import apply_device
m, n, k = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (4096, 4096, 192)
fast = os.environ.get("STRICT", "0") != "1"
A = torch.randn(n, m, dtype=torch.float64, device="cuda").t()
th = torch.rand(k, n - 1, dtype=torch.float64, device="cuda").t() * 6.283185307179586
C, S = torch.cos(th), torch.sin(th)
for _ in range(2):
    apply_device(A, (C, S), fast=fast)
torch.cuda.synchronize()
print("ok")
