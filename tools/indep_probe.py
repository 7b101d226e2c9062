"""Per-warp efficiency without chain coupling: one band (v1: k=8) or one band group
(g4: k=32) per tile, so every unit reads A and writes A and nothing waits on a peer."""
import sys, os, json, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, os
sys.path.insert(0, %r)
import torch
from paper_2412_01852_b200 import apply_device, flops_applied, _lib
for (m, n, k) in [(65536, 4096, int(os.environ["KK"])), (65536, 4096, 192)]:
    A = torch.randn(n, m, dtype=torch.float64, device="cuda").t()
    th = torch.rand(k, n - 1, dtype=torch.float64, device="cuda").t() * 6.283185307179586
    C, S = torch.cos(th), torch.sin(th)
    for _ in range(2): apply_device(A, (C, S), fast=True)
    torch.cuda.synchronize(); ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); apply_device(A, (C, S), fast=True); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(os.environ["RS_KERNEL"], m, n, k, "%%.3f ms %%.2f TF/s" %% (min(ts), flops_applied(m, n, k) / min(ts) / 1e9), _lib.plan_info(m, n, k), flush=True)
''' % ROOT
for var, kk in (("v1", "8"), ("g4", "32"), ("g2", "16")):
    subprocess.run([sys.executable, "-c", code], env=dict(os.environ, RS_KERNEL=var, KK=kk), timeout=600)
