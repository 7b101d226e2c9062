import sys, os, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2412_01852_b200 import apply_host, apply_cuda
m, n, k = 4096, 4096, 192
hA = torch.empty_strided((m, n), (1, m), dtype=torch.float64, pin_memory=True); hA.normal_()
th = np.random.default_rng(0).uniform(0, 2 * np.pi, (n - 1, k))
hC = torch.empty_strided((n - 1, k), (1, n - 1), dtype=torch.float64, pin_memory=True)
hS = torch.empty_strided((n - 1, k), (1, n - 1), dtype=torch.float64, pin_memory=True)
hC.copy_(torch.from_numpy(np.cos(th))); hS.copy_(torch.from_numpy(np.sin(th)))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
stream = torch.cuda.current_stream()
for name, fn in (("apply_host", lambda: apply_host(hA, (hC, hS), fast=True)), ("apply_cuda", lambda: apply_cuda(hA, (hC, hS), fast=True))):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    for fl in (False, True):
        ev, wall = [], []
        for _ in range(8):
            if fl: flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter(); e0.record(stream); fn(); e1.record(stream); torch.cuda.synchronize()
            wall.append((time.perf_counter() - t0) * 1e3); ev.append(e0.elapsed_time(e1))
        print(name, "flush" if fl else "noflush", "events %.3f ms wall %.3f ms" % (np.mean(ev), np.mean(wall)), flush=True)
