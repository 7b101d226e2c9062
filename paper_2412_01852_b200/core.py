"""Host-side mirror of the reference's rotation-sequence data model.

Same names, argument meaning and error behaviour as the reference package
``rotseq`` so that callers (and tests written against it) switch over unchanged:

* ``TransformKind``            /root/reference/pkg/src/rotseq/core.py:29-38
* ``require_colmajor``         core.py:41-51
* ``RotationSequence``         core.py:54-91
* ``generate_sequence``        core.py:94-107
* ``_check_apply_args``        core.py:110-117
* ``make_inputs``              verification.py:102-105

Extensions the reference does not define are explicit here:
``Side`` (right = column pairs, the reference's only side; left = row pairs,
xLASR SIDE='L') and ``Order`` (forward = the reference's order; reverse = each
sweep p still ascending, j descending, xLASR DIRECT='B' per sweep), plus fp32.
Nothing in this module touches a GPU.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field

import numpy as np


class TransformKind(enum.Enum):
    """2x2 action on a column pair (core.py:29-38).

    ROTATION is G = [[c, s], [-s, c]]; REFLECTOR is H = [[c, s], [s, -c]]
    evaluated with the 3-multiply / 3-addition scheme.
    """

    ROTATION = "rotation"
    REFLECTOR = "reflector"


class Side(enum.Enum):
    RIGHT = "right"   # A <- A * G: rotate column pairs (j, j+1); reference semantics
    LEFT = "left"     # A <- G^T * A: rotate row pairs (j, j+1)


class Order(enum.Enum):
    FORWARD = "forward"  # p ascending, j ascending (core.py:195-205)
    REVERSE = "reverse"  # p ascending, j descending within each sweep


SUPPORTED_DTYPES = (np.float64, np.float32)


def _as_enum(value, enum_cls, name):
    """Coerce ``value`` to ``enum_cls``. Accepts this package's enums, their string
    values, and any other enum whose ``.value`` is one of them — in particular the
    reference's own ``rotseq.TransformKind`` (core.py:29-38), so reference call sites
    pass their objects through unchanged."""
    if isinstance(value, enum_cls):
        return value
    raw = value.value if isinstance(value, enum.Enum) else value
    try:
        return enum_cls(raw)
    except ValueError:
        raise ValueError(f"{name} must be one of {[e.value for e in enum_cls]}, got {value!r}") from None


def is_sequence_object(seq) -> bool:
    """True for a rotation-sequence object: anything exposing ``C`` and ``S`` arrays
    (this package's ``RotationSequence`` or the reference's, core.py:54-91)."""
    return hasattr(seq, "C") and hasattr(seq, "S") and not isinstance(seq, (tuple, list))


def sequence_parts(seq):
    """(C, S, n_cols) of a sequence object or of a ``(C, S)`` pair.

    ``n_cols`` is the object's own ``n_cols`` when it has one (the reference's
    ``RotationSequence`` records it), else ``C.shape[0] + 1``."""
    if is_sequence_object(seq):
        C, S = seq.C, seq.S
        n_cols = getattr(seq, "n_cols", None)
        if n_cols is None:
            n_cols = int(C.shape[0]) + 1
        return C, S, int(n_cols)
    try:
        C, S = seq
    except (TypeError, ValueError):
        raise ValueError("seq must be a RotationSequence-like object (with .C/.S) or a (C, S) pair") from None
    return C, S, int(C.shape[0]) + 1


def require_colmajor(A: np.ndarray, name: str = "A", dtypes=(np.float64,)) -> None:
    """Validate a column-major matrix (core.py:41-51); views with ld > rows ok.

    The reference accepts float64 only; the B200 path additionally accepts
    float32 when ``dtypes`` says so (BASELINE config 4).
    """
    if not isinstance(A, np.ndarray) or A.ndim != 2:
        raise ValueError(f"{name} must be a 2-D numpy array")
    if A.dtype not in [np.dtype(d) for d in dtypes]:
        want = " or ".join(np.dtype(d).name for d in dtypes)
        raise ValueError(f"{name} must have dtype {want}, got {A.dtype}")
    if A.shape[0] > 1 and A.strides[0] != A.itemsize:
        raise ValueError(
            f"{name} must be column-major (order='F' or a row block of an "
            "F-ordered array); use np.asfortranarray"
        )


@dataclass(frozen=True)
class RotationSequence:
    """k sequences of n-1 transforms acting on an n-column matrix (core.py:54-91).

    ``C`` and ``S`` have shape ``(n_cols - 1, k)`` in column-major layout.
    ``orthonormal`` records whether c^2 + s^2 = 1 was verified.
    """

    n_cols: int
    k: int
    C: np.ndarray = field(repr=False)
    S: np.ndarray = field(repr=False)
    orthonormal: bool = True

    ORTHONORMAL_TOL = 1e-12

    @classmethod
    def from_arrays(cls, C, S, check_orthonormal: bool = True) -> "RotationSequence":
        C = np.asfortranarray(C, dtype=np.float64)
        S = np.asfortranarray(S, dtype=np.float64)
        if C.ndim != 2 or C.shape != S.shape:
            raise ValueError(f"C and S must share a 2-D shape, got {C.shape} vs {S.shape}")
        rows, k = C.shape
        if rows < 1 or k < 1:
            raise ValueError("sequence needs at least one rotation row and one sequence")
        err = float(np.abs(C * C + S * S - 1.0).max())
        if check_orthonormal and err > cls.ORTHONORMAL_TOL:
            raise ValueError(
                f"c^2 + s^2 deviates from 1 by {err:.3e} (> {cls.ORTHONORMAL_TOL}); "
                "pass check_orthonormal=False to accept non-orthonormal input"
            )
        return cls(n_cols=rows + 1, k=k, C=C, S=S, orthonormal=err <= cls.ORTHONORMAL_TOL)


def generate_sequence(n: int, k: int, seed: int) -> RotationSequence:
    """Deterministic random orthonormal sequence (core.py:94-107): angles uniform
    on [0, 2*pi) from Philox(seed), C = cos, S = sin."""
    if n < 2:
        raise ValueError(f"need n >= 2 columns, got {n}")
    if k < 1:
        raise ValueError(f"need k >= 1 sequences, got {k}")
    rng = np.random.Generator(np.random.Philox(seed))
    theta = rng.uniform(0.0, 2.0 * np.pi, size=(n - 1, k))
    return RotationSequence.from_arrays(np.cos(theta), np.sin(theta))


def make_inputs(m: int, n: int, k: int, seed: int) -> tuple[np.ndarray, RotationSequence]:
    """A = Philox(seed) standard normal (F-order), sequence from seed+1
    (verification.py:102-105)."""
    rng = np.random.Generator(np.random.Philox(seed))
    A = np.asfortranarray(rng.standard_normal((m, n)))
    return A, generate_sequence(n, k, seed + 1)


def rotated_length(shape, side: Side) -> int:
    return shape[0] if side is Side.LEFT else shape[1]


def check_apply_args(A: np.ndarray, seq, side: Side = Side.RIGHT,
                     dtypes=(np.float64,)) -> None:
    """_check_apply_args (core.py:110-117), generalised to the left side. ``seq`` is
    a sequence object (ours or the reference's) or a ``(C, S)`` pair."""
    require_colmajor(A, dtypes=dtypes)
    n_cols = sequence_parts(seq)[2]
    if side is Side.RIGHT:
        if A.shape[1] < 2:
            raise ValueError(f"matrix needs at least 2 columns, got {A.shape[1]}")
        if n_cols != A.shape[1]:
            raise ValueError(f"sequence acts on {n_cols} columns but matrix has {A.shape[1]}")
    else:
        if A.shape[0] < 2:
            raise ValueError(f"matrix needs at least 2 rows for left-side application, got {A.shape[0]}")
        if n_cols != A.shape[0]:
            raise ValueError(f"sequence acts on {n_cols} rows but matrix has {A.shape[0]}")


def flops_applied(m: int, n: int, k: int, side: Side = Side.RIGHT) -> float:
    """6 flops per rotation element (model.py:123-126): 6*m*(n-1)*k on the right,
    6*n*(m-1)*k on the left."""
    if side is Side.LEFT:
        return 6.0 * n * max(m - 1, 0) * k
    return 6.0 * m * max(n - 1, 0) * k
