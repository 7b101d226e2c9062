"""Dispatch point and equivalence grids (mirror of rotseq.verification).

``run_variant`` keeps the reference's role as "the single dispatch point for
every algorithm" (verification.py:3-6, 50-85) and its signature (``plan``,
``shape``, ``n_r``, ``k_r``, ``threads`` accepted and ignored: CPU cache and thread
knobs). The B200 build registers its own algorithms under new names, exactly as a
new backend would be added to the reference's ``ALGORITHMS`` tuple
(verification.py:42):

* ``cuda``        the register-window band pipeline (product path)
* ``cuda-naive``  one thread per row, plain sweep loop (independent GPU check)

``ROTSEQ_PERTURB_KERNEL=1`` injects a one-ulp perturbation into the output of the
algorithm under test (``cuda``, the kernel path), as the reference does for its kernel
tiers (verification.py:8-11, 40-47, 76, 83); the checking algorithm (``cuda-naive``)
is never perturbed, so the verifier's failure path can itself be tested.

The grids mirror ``bitwise_grid`` / ``oracle_grid`` (verification.py:181-219). The
explicit-Q chain accumulates Q on the host (``accumulate_q``, the reference's
oracle.py:102-109, with the 2x2 formulas of core.py:130-149 evaluated by numpy on
whole columns) and multiplies in float64 — it shares no code with the CUDA kernels.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from .apply import apply_cuda
from .compare import ComparisonReport, compare
from .core import Order, RotationSequence, Side, TransformKind, _as_enum, make_inputs, sequence_parts

FAULT_ENV = "ROTSEQ_PERTURB_KERNEL"

ALGORITHMS = ("cuda", "cuda-naive")
KERNEL_ALGORITHMS = ("cuda",)  # outputs subject to the fault-injection hook


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
    plan=None,
    shape=None,
    n_r: int = 2,
    k_r: int = 2,
    threads: int = 1,
    *,
    side: Side = Side.RIGHT,
    order: Order = Order.FORWARD,
) -> None:
    """Apply one named algorithm to A in place (verification.py:50-85).

    Same positional signature as the reference; ``seq`` and ``kind`` may be the
    reference's own objects. ``side``/``order`` (keyword-only) are this build's
    extensions."""
    if threads < 1:
        raise ValueError(f"threads must be >= 1, got {threads}")
    if algo == "cuda":
        apply_cuda(A, seq, kind=kind, fast=fast, side=side, order=order, algo="pipeline")
        _maybe_perturb(A)
    elif algo == "cuda-naive":
        apply_cuda(A, seq, kind=kind, fast=fast, side=side, order=order, algo="naive")
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


@dataclass(frozen=True)
class CaseResult:
    """One grid case (verification.py:110-128)."""

    algo: str
    config: str
    kind: str
    m: int
    n: int
    k: int
    report: ComparisonReport

    @property
    def ok(self) -> bool:
        return bool(self.report.passed)

    def __str__(self):
        return f"{self.algo:10s} [{self.config}] {self.kind} m={self.m} n={self.n} k={self.k}: {self.report}"


def accumulate_q(seq, kind=TransformKind.ROTATION) -> np.ndarray:
    """Explicit n x n matrix Q with (sequence applied to A) == A @ Q, accumulated on the
    host from the identity in plain order (p outer, j inner: core.py:195-205) with the
    reference's 2x2 formulas (core.py:130-149) on whole columns. Reference:
    ``accumulate_q`` (oracle.py:102-109)."""
    kind = _as_enum(kind, TransformKind, "kind")
    C, S, n = sequence_parts(seq)
    C = np.asarray(C, dtype=np.float64)
    S = np.asarray(S, dtype=np.float64)
    Q = np.eye(n, order="F")
    for p in range(C.shape[1]):
        for j in range(n - 1):
            c, s = C[j, p], S[j, p]
            x, y = Q[:, j].copy(), Q[:, j + 1].copy()
            if kind is TransformKind.REFLECTOR:
                w = s * (x + y)
                Q[:, j] = w + (c - s) * x
                Q[:, j + 1] = w - (c + s) * y
            else:
                Q[:, j] = c * x + s * y
                Q[:, j + 1] = c * y - s * x
    return Q


def bitwise_grid(kind, quick: bool = False, seed: int = 7, algo: str = "cuda"):
    """Criterion 1 (verification.py:181-195): ``algo`` in strict arithmetic,
    bit-identical to the independent plain-loop GPU kernel (``cuda-naive``)."""
    kind = _as_enum(kind, TransformKind, "kind")
    for m, n, k in case_grid(quick):
        A0, seq = make_inputs(m, n, k, seed)
        ref = A0.copy(order="F")
        run_variant("cuda-naive", ref, seq, kind, fast=False)
        got = A0.copy(order="F")
        run_variant(algo, got, seq, kind, fast=False)
        yield CaseResult(algo, "vs cuda-naive", kind.value, m, n, k, compare(ref, got, tol_profile="strict"))


def oracle_grid(kind, seed: int = 11, algos=ALGORITHMS):
    """Criterion 2 (verification.py:198-219): every algorithm against A0 @ Q with Q
    accumulated on the host; Frobenius-relative tolerance 1e-12 (rotations) or 1e-11
    (reflectors), as in the reference."""
    kind = _as_enum(kind, TransformKind, "kind")
    tol = 1e-12 if kind is TransformKind.ROTATION else 1e-11
    for mn in (16, 48, 96):
        for k in (3, 18):
            A0, seq = make_inputs(mn, mn, k, seed)
            expected = np.asfortranarray(A0 @ accumulate_q(seq, kind))
            for algo in algos:
                got = A0.copy(order="F")
                run_variant(algo, got, seq, kind, fast=False)
                rep = compare(expected, got)
                rep = ComparisonReport(max_abs_diff=rep.max_abs_diff, max_rel_diff=rep.max_rel_diff,
                                       frobenius_rel_diff=rep.frobenius_rel_diff,
                                       bitwise_equal=rep.bitwise_equal, passed=rep.frobenius_rel_diff <= tol)
                yield CaseResult(algo, "explicit Q", kind.value, mn, mn, k, rep)
