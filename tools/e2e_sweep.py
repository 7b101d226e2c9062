"""rs_apply_host timing sweep over streaming chunk/group sizes (developer tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2412_01852_b200 import apply_host
m = n = 4096; k = 192
hA = torch.empty_strided((m, n), (1, m), dtype=torch.float64, pin_memory=True); hA.normal_()
th = np.random.default_rng(0).uniform(0, 2 * np.pi, (n - 1, k))
hC = torch.from_numpy(np.asfortranarray(np.cos(th))).pin_memory()
hS = torch.from_numpy(np.asfortranarray(np.sin(th))).pin_memory()
configs = [c.split(":") for c in (sys.argv[1:] or ["8:1", "8:8", "16:4", "64:4", "64:8"])]
res = {tuple(c): [] for c in configs}
for rep in range(int(os.environ.get('REPS', '4'))):
    for c in configs:
        os.environ["RS_HOST_CHUNKS"], os.environ["RS_HOST_GROUP"] = c
        apply_host(hA, (hC, hS), fast=True)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5):
            apply_host(hA, (hC, hS), fast=True)
        res[tuple(c)].append((time.perf_counter() - t) / 5 * 1e3)
for c, v in res.items():
    print(f"chunks {c[0]:>3} group {c[1]:>2}: min {min(v):.3f} ms  median {sorted(v)[len(v)//2]:.3f} ms")
