"""Developer timing probe: kernel-only timing of chosen BASELINE configs.
Usage: [RS_LIB_PATH=...] python tools/qb.py c2 c3 c4 c5 c1 [reps]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_01852_b200 import apply_device, flops_applied, Side, _lib

CFG = {"c1": (512, 512, 64, torch.float64, "right", "forward"),
       "c2": (4096, 4096, 192, torch.float64, "right", "forward"),
       "c3": (65536, 2048, 256, torch.float64, "right", "forward"),
       "c3s": (8192, 2048, 256, torch.float64, "right", "forward"),
       "c4": (8192, 8192, 128, torch.float32, "right", "forward"),
       "c5": (16384, 16384, 96, torch.float64, "left", "reverse")}


def bench(name, reps):
    m, n, k, dtype, side, order = CFG[name]
    dev = torch.device("cuda")
    A = torch.randn(n, m, dtype=dtype, device=dev).t()
    length = m if side == "left" else n
    th = torch.rand(k, length - 1, dtype=torch.float64, device=dev).t() * 6.283185307179586
    C, S = torch.cos(th).to(dtype), torch.sin(th).to(dtype)
    for _ in range(3):
        apply_device(A, (C, S), fast=True, side=side, order=order)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); apply_device(A, (C, S), fast=True, side=side, order=order); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    f = flops_applied(m, n, k, Side(side))
    ts.sort()
    info = _lib.plan_info(m, n, k, 1 if side == "left" else 0, 0, 0 if dtype == torch.float64 else 1)
    print(f"{os.environ.get('RS_LIB_PATH', 'default').split('/')[-1]:>12} {info['grid_ctas']}x{info['warps_per_cta']}w u={info['units']} {name}: best {ts[0]:.4f} ms median {ts[len(ts)//2]:.4f} ms"
          f" -> {f/ts[0]/1e9:.2f} / {f/ts[len(ts)//2]/1e9:.2f} TF/s (step incl. pack)", flush=True)


for a in sys.argv[1:]:
    if a.count("x") == 2 and a.replace("x", "").isdigit():
        mm, nn, kk = (int(v) for v in a.split("x"))
        CFG[a] = (mm, nn, kk, torch.float64, "right", "forward")
names = [a for a in sys.argv[1:] if a in CFG]
reps = next((int(a) for a in sys.argv[1:] if a.isdigit()), 20)
for nm in names or ["c2"]:
    bench(nm, reps)
