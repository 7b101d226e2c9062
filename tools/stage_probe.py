import sys, os, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
code = r'''
import sys, os
sys.path.insert(0, "%s")
import torch
from paper_2412_01852_b200 import apply_device, flops_applied, _lib
for (m, n, k) in [(4096, 4096, 192), (65536, 2048, 256), (16384, 4096, 192)]:
    A = torch.randn(n, m, dtype=torch.float64, device="cuda").t()
    th = torch.rand(k, n - 1, dtype=torch.float64, device="cuda").t() * 6.283185307179586
    C, S = torch.cos(th), torch.sin(th)
    for _ in range(2): apply_device(A, (C, S), fast=True)
    torch.cuda.synchronize(); ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); apply_device(A, (C, S), fast=True); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(os.environ.get("RS_LIB_PATH","").split("/")[-1], m, n, k, "%%.3f ms %%.2f TF/s" %% (min(ts), flops_applied(m, n, k) / min(ts) / 1e9), _lib.plan_info(m, n, k)["warps_per_cta"], flush=True)
''' % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for lib in sorted(os.listdir(os.path.join(os.path.dirname(os.path.abspath(__file__)), "exp"))):
    env = dict(os.environ, RS_LIB_PATH=os.path.join(os.path.dirname(os.path.abspath(__file__)), "exp", lib))
    subprocess.run([sys.executable, "-c", code], env=env, timeout=300)
