"""Quick GPU parity probe (developer tool): pipeline/naive vs the CPU oracle."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2412_01852_b200 import make_inputs, generate_sequence, apply_cuda, compare
from oracle import oracle

def run(m, n, k, seed=7, side="right", order="forward", kind="rotation", fast=False, algo="pipeline"):
    A0, seq = make_inputs(m, n, k, seed)
    C, S = seq.C, seq.S
    if side == "left":
        s2 = generate_sequence(m, k, seed + 2); C, S = s2.C, s2.S
    ref = A0.copy(order="F")
    oracle.apply_naive(ref, C, S, side=side, order=order, kind=kind)
    got = A0.copy(order="F")
    apply_cuda(got, (C, S), kind=kind, fast=fast, side=side, order=order, algo=algo)
    rep = compare(ref, got, "strict" if not fast else "fast", k=k)
    print(f"{algo:8s} m={m:5d} n={n:5d} k={k:4d} {side:5s} {order:7s} {kind:9s} fast={fast}: {rep}", flush=True)
    return rep.passed

ok = True
for algo in ("naive", "pipeline"):
    for (m, n, k) in [(3, 9, 3), (32, 64, 8), (33, 40, 9), (64, 64, 12), (129, 64, 5), (257, 33, 12), (100, 300, 64), (70, 17, 30), (31, 3, 7), (1, 2, 1)]:
        ok &= run(m, n, k, algo=algo)
for side in ("right", "left"):
    for order in ("forward", "reverse"):
        for kind in ("rotation", "reflector"):
            ok &= run(65, 70, 17, side=side, order=order, kind=kind)
            ok &= run(65, 70, 17, side=side, order=order, kind=kind, fast=True)
ok &= run(4096, 512, 64)
# forced multi-round / multi-CTA geometries (exercise ring, flag and reorder paths)
for mw, grid in [("1", "1"), ("2", "3"), ("3", "2"), ("4", "5"), ("5", "7"), ("2", "")]:
    os.environ["RS_DEBUG_MAX_WARPS"] = mw
    if grid: os.environ["RS_DEBUG_GRID"] = grid
    else: os.environ.pop("RS_DEBUG_GRID", None)
    print("RS_DEBUG_MAX_WARPS", mw, "RS_DEBUG_GRID", grid)
    for (m, n, k) in [(100, 50, 40), (300, 37, 33), (64, 200, 70), (33, 9, 24)]:
        ok &= run(m, n, k)
    ok &= run(90, 60, 41, side="left", order="reverse", kind="reflector")
os.environ.pop("RS_DEBUG_MAX_WARPS", None); os.environ.pop("RS_DEBUG_GRID", None)
ok &= run(65536 // 8, 2048, 256)
print("ALL OK" if ok else "FAILURES")
