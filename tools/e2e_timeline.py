"""rs_apply_host timeline for a few chunk/group settings (developer tool)."""
import sys, os, time, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
code = r'''
import sys, os, time
sys.path.insert(0, %r)
import numpy as np, torch
from paper_2412_01852_b200 import apply_host
m, n, k = 4096, 4096, 192
hA = torch.empty_strided((m, n), (1, m), dtype=torch.float64, pin_memory=True); hA.normal_()
th = np.random.default_rng(0).uniform(0, 2 * np.pi, (n - 1, k))
hC = torch.empty_strided((n - 1, k), (1, n - 1), dtype=torch.float64, pin_memory=True)
hS = torch.empty_strided((n - 1, k), (1, n - 1), dtype=torch.float64, pin_memory=True)
hC.copy_(torch.from_numpy(np.cos(th))); hS.copy_(torch.from_numpy(np.sin(th)))
for _ in range(3): apply_host(hA, (hC, hS), fast=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5): apply_host(hA, (hC, hS), fast=True)
torch.cuda.synchronize()
print(os.environ.get("TAG"), "%%.3f ms" %% ((time.perf_counter() - t0) / 5 * 1e3), flush=True)
if os.environ.get("DBG"):
    os.environ["RS_HOST_DEBUG"] = "1"
    apply_host(hA, (hC, hS), fast=True); torch.cuda.synchronize()
''' % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for tag in sys.argv[1:]:
    env = dict(os.environ, TAG=tag)
    for kv in tag.split(","):
        if "=" in kv:
            a, b = kv.split("=", 1); env[a] = b
    subprocess.run([sys.executable, "-c", code], env=env, timeout=300)
