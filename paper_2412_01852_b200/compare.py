"""Tolerance profiles and comparison reports (mirror of rotseq.oracle:23-99).

Attribution: ``ComparisonReport`` (including ``__str__``) and the body of
``compare`` are copied, nearly verbatim, from the reference's
``/root/reference/pkg/src/rotseq/oracle.py:23-99``. They are the tolerance contract
every test in both packages agrees on, so they are kept identical on purpose.

``compare`` and the profiles carry the reference's meaning of "equal":
strict = bitwise; fast = Frobenius-relative and row-scaled elementwise error
<= 16*k*eps (oracle.py:26-29, 82-90). ``baseline_tol`` is BASELINE.json's
acceptance bound ||A_gpu - A_ref||_F / ||A_ref||_F <= 10*k*eps(dtype).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

EPS = float(np.finfo(np.float64).eps)
EPS32 = float(np.finfo(np.float32).eps)


def fast_mode_tol(k: int, eps: float = EPS) -> float:
    return 16.0 * max(k, 1) * eps


def norm_preservation_tol(k: int, eps: float = EPS) -> float:
    return 100.0 * max(k, 1) * eps


def baseline_tol(k: int, dtype=np.float64) -> float:
    """BASELINE.json parity bound: 10*k*eps of the working dtype."""
    return 10.0 * max(k, 1) * float(np.finfo(np.dtype(dtype)).eps)


@dataclass(frozen=True)
class ComparisonReport:
    max_abs_diff: float
    max_rel_diff: float
    frobenius_rel_diff: float
    bitwise_equal: bool
    passed: bool | None = None

    def __str__(self):
        verdict = "" if self.passed is None else ("  PASS" if self.passed else "  FAIL")
        return (
            f"max|d|={self.max_abs_diff:.3e} rel={self.max_rel_diff:.3e} "
            f"fro={self.frobenius_rel_diff:.3e} bitwise={self.bitwise_equal}{verdict}"
        )


def _bits(X: np.ndarray) -> np.ndarray:
    X = np.ascontiguousarray(X)
    return X.view(np.uint64 if X.dtype == np.float64 else np.uint32)


def compare(X, Y, tol_profile: str | None = None, k: int = 1) -> ComparisonReport:
    """Elementwise comparison (oracle.py:54-99). Profiles: None, 'strict'
    (bitwise), 'fast' (16*k*eps), 'baseline' (10*k*eps Frobenius)."""
    X = np.asarray(X)
    Y = np.asarray(Y)
    if X.shape != Y.shape:
        raise ValueError(f"shape mismatch: {X.shape} vs {Y.shape}")
    bitwise = X.dtype == Y.dtype and bool(np.array_equal(_bits(X), _bits(Y)))
    Xd = X.astype(np.float64)
    Yd = Y.astype(np.float64)
    diff = np.abs(Xd - Yd)
    max_abs = float(diff.max()) if diff.size else 0.0
    scale = np.maximum(np.abs(Xd), np.abs(Yd))
    with np.errstate(invalid="ignore", divide="ignore"):
        rel = np.where(diff > 0, diff / np.maximum(scale, np.finfo(np.float64).tiny), 0.0)
    max_rel = float(rel.max()) if rel.size else 0.0
    x_fro = float(np.linalg.norm(Xd))
    fro_rel = float(np.linalg.norm(Xd - Yd)) / (x_fro if x_fro > 0 else 1.0)
    passed = None
    eps = EPS if X.dtype == np.float64 else EPS32
    if tol_profile == "strict":
        passed = bitwise
    elif tol_profile == "fast":
        tol = fast_mode_tol(k, eps)
        if Xd.ndim == 2 and Xd.size:
            row_norms = np.linalg.norm(Xd, axis=1, keepdims=True)
            elem_ok = bool(np.all(diff <= tol * np.maximum(row_norms, np.finfo(np.float64).tiny)))
        else:
            elem_ok = max_abs <= tol
        passed = fro_rel <= tol and elem_ok
    elif tol_profile == "baseline":
        passed = fro_rel <= 10.0 * max(k, 1) * eps
    elif tol_profile is not None:
        raise ValueError(f"unknown tolerance profile {tol_profile!r}")
    return ComparisonReport(max_abs, max_rel, fro_rel, bitwise, passed)
