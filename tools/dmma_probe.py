"""Time the FP64 tensor-core variant (rs_apply_dmma_f64) against the pipeline kernel on the
BASELINE fp64 right-side shapes (device-resident, CUDA events, best of reps).
Usage: python tools/dmma_probe.py [m n k ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2412_01852_b200 import PackedSequence, apply_dmma, dmma_workspace_bytes, flops_applied  # noqa: E402

args = [int(x) for x in sys.argv[1:]] or [4096, 4096, 192, 8192, 2048, 256, 65536, 2048, 256]
for i in range(0, len(args), 3):
    m, n, k = args[i:i + 3]
    A = torch.randn(n, m, dtype=torch.float64, device="cuda").t()
    th = torch.rand(k, n - 1, dtype=torch.float64, device="cuda").t() * 6.283185307179586
    C, S = torch.cos(th), torch.sin(th)
    ws = torch.empty(dmma_workspace_bytes(m, n, k), dtype=torch.uint8, device="cuda")
    ps = PackedSequence((C, S), A.shape, fast_only=True)
    f = flops_applied(m, n, k)
    out = []
    for name, fn in (("dmma", lambda: apply_dmma(A, (C, S), workspace=ws)), ("pipeline", lambda: ps.apply(A, fast=True))):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out.append(f"{name} {best:.3f} ms {f / best / 1e9:.2f} TF/s")
    print(f"{m}x{n} k={k}: " + " | ".join(out), flush=True)
