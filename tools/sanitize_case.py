"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck), one tool per run:

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_case.py
    RS_DEBUG_GRID=1 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_case.py

Covers the pipeline kernel in forced multi-round / multi-CTA geometries (ring hand-offs,
progress flags through A, tail-first CTA order), both sides and orders, strict, fast
(scaled) and fast with a per-unit fallback, the host-streaming entry point, the packed
mode and the micro-kernel API; every result is checked against the CPU oracle (exit 1 on
a mismatch), so a sanitizer report and a wrong answer are both visible.
"""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main() -> int:
    import torch

    from oracle import oracle
    from paper_2412_01852_b200 import apply_cuda, compare, generate_sequence, make_inputs
    from paper_2412_01852_b200.kernels import KernelShape, kernel_wave_apply

    oracle.build()
    torch.cuda.set_device(0)
    bad = 0
    geoms = [("1", ""), ("4", "3"), ("2", "")] if not os.environ.get("RS_DEBUG_GRID") else [("1", None), ("4", None)]
    cases = [(100, 50, 40, "right", "forward", "rotation"), (90, 60, 41, "left", "reverse", "reflector"),
             (129, 130, 20, "left", "forward", "rotation"), (300, 37, 33, "right", "reverse", "reflector")]
    for mw, grid in geoms:
        os.environ["RS_DEBUG_MAX_WARPS"] = mw
        if grid is not None:
            if grid:
                os.environ["RS_DEBUG_GRID"] = grid
            else:
                os.environ.pop("RS_DEBUG_GRID", None)
        for (m, n, k, side, order, kind) in cases:
            A0, seq = make_inputs(m, n, k, 2)
            if side == "left":
                seq = generate_sequence(m, k, 3)
            C, S = seq.C.copy(order="F"), seq.S.copy(order="F")
            C[3, 1], S[3, 1] = 0.0, 1.0  # one exact swap: a per-unit fallback in fast mode
            ref = A0.copy(order="F")
            oracle.apply_naive(ref, C, S, side=side, order=order, kind=kind)
            for fast in (False, True):
                dA = torch.from_numpy(A0.copy(order="F")).cuda()
                apply_cuda(dA, (C, S), kind=kind, fast=fast, side=side, order=order)
                got = dA.cpu().numpy()
                rep = compare(ref, got, "baseline" if fast else "strict", k=k)
                if not rep.passed:
                    bad += 1
                    print(f"MISMATCH device mw={mw} grid={grid} {m}x{n} k={k} {side}/{order}/{kind} fast={fast}: {rep}")
            # host-streaming entry point (copy-in / compute / copy-out overlap)
            got = A0.copy(order="F")
            apply_cuda(got, (C, S), kind=kind, fast=False, side=side, order=order)
            if not compare(ref, got, "strict").passed:
                bad += 1
                print(f"MISMATCH host mw={mw} grid={grid} {m}x{n} k={k} {side}/{order}/{kind}")
    # micro-kernel API
    rng = np.random.Generator(np.random.Philox(5))
    for k_r in (1, 3, 8, 11):
        P0 = np.ascontiguousarray(rng.standard_normal((40, 33)))
        th = rng.uniform(0, 2 * np.pi, size=20 * k_r)
        ref = P0.copy()
        oracle.wave_apply(ref, np.cos(th), np.sin(th), 20, k_r, 2)
        got = P0.copy()
        kernel_wave_apply(got, np.cos(th), np.sin(th), 20, KernelShape(33, k_r), "rotation", 2)
        if not compare(ref, got, "strict").passed:
            bad += 1
            print(f"MISMATCH wave k_r={k_r}")
    torch.cuda.synchronize()
    print(f"sanitize cases done: {bad} mismatches")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
