"""Developer timing probe: device-resident apply on a BASELINE config."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2412_01852_b200 import apply_device, flops_applied, _lib

def bench(m, n, k, dtype=torch.float64, fast=True, side="right", order="forward", reps=5):
    dev = torch.device("cuda")
    A = torch.randn(n, m, dtype=dtype, device=dev).t()  # column-major view m x n
    length = m if side == "left" else n
    th = torch.rand(k, length - 1, dtype=torch.float64, device=dev).t() * 6.283185307179586
    C, S = torch.cos(th).to(dtype), torch.sin(th).to(dtype)
    for _ in range(2):
        apply_device(A, (C, S), fast=fast, side=side, order=order)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); apply_device(A, (C, S), fast=fast, side=side, order=order); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    f = flops_applied(m, n, k, __import__("paper_2412_01852_b200").Side(side))
    t = min(ts)
    info = _lib.plan_info(m, n, k, 1 if side == "left" else 0, 0, 0 if dtype == torch.float64 else 1)
    print(f"m={m} n={n} k={k} {dtype} fast={fast} {side}/{order}: best {t:.3f} ms median {sorted(ts)[len(ts)//2]:.3f} ms "
          f"-> {f/t/1e9:.2f} TF/s  plan={info}", flush=True)

bench(4096, 4096, 192)
bench(4096, 4096, 192, fast=False)
bench(512, 512, 64)
bench(65536, 2048, 256)
bench(8192, 8192, 128, dtype=torch.float32)
bench(16384, 16384, 96, side="left", order="reverse")
