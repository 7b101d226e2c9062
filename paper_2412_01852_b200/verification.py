"""Dispatch point and equivalence grids (mirror of rotseq.verification).

``run_variant`` keeps the reference's role as "the single dispatch point for
every algorithm" (verification.py:3-6, 50-85). The B200 build registers its
own algorithms under new names, exactly as a new backend would be added to the
reference's ``ALGORITHMS`` tuple (verification.py:42):

* ``cuda``        the register-window band pipeline (product path)
* ``cuda-naive``  one thread per row, plain sweep loop (independent GPU check)

``ROTSEQ_PERTURB_KERNEL=1`` injects a one-ulp perturbation into the output of
the kernel paths, as the reference does (verification.py:8-11, 40-47), so the
verifier's failure path can itself be tested.
"""

from __future__ import annotations

import os

import numpy as np

from .apply import apply_cuda
from .core import Order, RotationSequence, Side, TransformKind

FAULT_ENV = "ROTSEQ_PERTURB_KERNEL"

ALGORITHMS = ("cuda", "cuda-naive")


def _maybe_perturb(A) -> None:
    if not os.environ.get(FAULT_ENV):
        return
    if isinstance(A, np.ndarray):
        if A.size:
            A.flat[0] = np.nextafter(A.flat[0], np.inf)
        return
    import torch  # noqa: PLC0415

    if A.numel():
        v = A[0, 0].item()
        A[0, 0] = float(np.nextafter(np.array(v, dtype=np.float64 if A.dtype == torch.float64 else np.float32),
                                     np.inf))


def run_variant(
    algo: str,
    A,
    seq: RotationSequence,
    kind: TransformKind = TransformKind.ROTATION,
    fast: bool = False,
    side: Side = Side.RIGHT,
    order: Order = Order.FORWARD,
    **_cpu_knobs,
) -> None:
    """Apply one named algorithm to A in place (verification.py:50-85).

    The reference's CPU-only keyword arguments (plan, shape, n_r, k_r, threads)
    are accepted and ignored so call sites port unchanged."""
    if algo == "cuda":
        apply_cuda(A, seq, kind=kind, fast=fast, side=side, order=order, algo="pipeline")
        _maybe_perturb(A)
    elif algo == "cuda-naive":
        apply_cuda(A, seq, kind=kind, fast=fast, side=side, order=order, algo="naive")
        _maybe_perturb(A)
    else:
        raise ValueError(f"unknown algorithm {algo!r}; choose from {ALGORITHMS}")


def case_grid(quick: bool = False):
    """(m, n, k) grid of the reference's criterion-1 check (verification.py:161-178)."""
    if quick:
        ms = (3, 17, 64)
        ns = (9, 33, 64)
        ks = (1, 3, 8)
    else:
        ms = (2, 3, 8, 17, 32, 33, 64, 129, 257)
        ns = (4, 9, 16, 33, 64, 128, 256)
        ks = (1, 2, 3, 5, 8, 12)
    for m in ms:
        for n in ns:
            seen = set()
            for k in ks:
                k = min(k, n - 1)
                if k in seen:
                    continue
                seen.add(k)
                yield m, n, k
