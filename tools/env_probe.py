"""Time configs under different env settings (each in a fresh process)."""
import sys, os, subprocess, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, os, json
sys.path.insert(0, %r)
import torch
from paper_2412_01852_b200 import apply_device, flops_applied, Side
cases = json.loads(os.environ["CASES"])
for (m, n, k, dt, side, order) in cases:
    dtype = torch.float64 if dt == "f64" else torch.float32
    A = torch.randn(n, m, dtype=dtype, device="cuda").t()
    ln = m if side == "left" else n
    th = torch.rand(k, ln - 1, dtype=torch.float64, device="cuda").t() * 6.283185307179586
    C, S = torch.cos(th).to(dtype), torch.sin(th).to(dtype)
    for _ in range(2): apply_device(A, (C, S), fast=True, side=side, order=order)
    torch.cuda.synchronize(); ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); apply_device(A, (C, S), fast=True, side=side, order=order); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    f = flops_applied(m, n, k, Side(side))
    print(os.environ.get("TAG",""), m, n, k, dt, side, order, "%%.3f ms %%.2f TF/s" %% (min(ts), f / min(ts) / 1e9), flush=True)
''' % ROOT
CASES = [(4096, 4096, 192, "f64", "right", "forward"), (65536, 2048, 256, "f64", "right", "forward"),
         (8192, 8192, 128, "f32", "right", "forward"), (16384, 16384, 96, "f64", "left", "reverse"),
         (8192, 2048, 256, "f64", "right", "forward")]
for tag in sys.argv[1:]:
    env = dict(os.environ, CASES=json.dumps(CASES), TAG=tag)
    for kv in tag.split(","):
        if "=" in kv:
            k, v = kv.split("=", 1); env[k] = v
    subprocess.run([sys.executable, "-c", code], env=env, timeout=600)
