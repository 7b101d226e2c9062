import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_01852_b200 import apply_device, flops_applied
def t(m, n, k, reps=5, **kw):
    A = torch.randn(n, m, dtype=torch.float64, device="cuda").t()
    th = torch.rand(k, n - 1, dtype=torch.float64, device="cuda").t() * 6.283185307179586
    C, S = torch.cos(th), torch.sin(th)
    for _ in range(2): apply_device(A, (C, S), fast=True)
    torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); apply_device(A, (C, S), fast=True); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return min(ts), flops_applied(m, n, k) / min(ts) / 1e9
for env in ["0", "1"]:
    os.environ["RS_DEBUG_NO_CHAIN"] = env
    for (m, n, k) in [(4096, 4096, 192), (65536, 2048, 256), (4096 * 4, 4096, 192)]:
        ms, tf = t(m, n, k)
        print(f"no_chain={env} m={m} n={n} k={k}: {ms:.3f} ms {tf:.2f} TF/s", flush=True)
