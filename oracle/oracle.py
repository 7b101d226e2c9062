"""CPU oracle for the rotation-sequence path — TEST INFRASTRUCTURE ONLY.

Restates the reference algorithm (package ``rotseq``, /root/reference/pkg/src/rotseq)
so the CUDA path can be checked without the reference being present (it is not on
the GPU box). Two independent restatements:

* ``numpy_apply_naive``  pure numpy, vectorised over rows; plain IEEE mul/add
  exactly as ``_naive_py`` + ``_rot_cols``/``_refl_cols`` (core.py:130-149, 195-205).
* ``apply_naive`` / ``apply_blocked`` in C (oracle/rotseq_oracle.c, built by
  ``make -C oracle``): the naive loop and the "kernel" tier
  (blocking.py:342-397, 420-476), strict and fast builds.

Both are pinned bit-for-bit to the reference by tests/test_oracle_golden.py
against fixtures the reference itself produced (tests/golden/make_golden.py).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may import
this module; the product package never does.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "librotseq_oracle.so")

_lib = None

# CacheSpec defaults (blocking.py:45-50) and the default kernel shape (128, 4)
# (verification.py:90-95) give this plan via choose_block_sizes (blocking.py:115-147).
DEFAULT_MR, DEFAULT_KR = 128, 4


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(
        os.path.join(HERE, "rotseq_oracle.c")
    ):
        subprocess.run(["make", "-s", "-C", HERE, "-B" if force else "all"], check=True)
    return LIB_PATH


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        lib = ctypes.CDLL(LIB_PATH)
        i64, i32, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        for suf in ("strict", "fast"):
            f = getattr(lib, f"oracle_apply_naive_f64_{suf}")
            f.restype = None
            f.argtypes = [vp, i64, i64, i64, vp, vp, i64, i64, i32, i32, i32, i64, i64]
            g = getattr(lib, f"oracle_apply_blocked_f64_{suf}")
            g.restype = i32
            g.argtypes = [vp, i64, i64, i64, vp, vp, i64, i64, i32, i64, i64, i64, i64, i64, i32]
            h = getattr(lib, f"oracle_partition_rows_{suf}")
            h.restype = None
            h.argtypes = [i64, i64, i64, vp]
        _lib = lib
    return _lib


def _check_A(A):
    if not isinstance(A, np.ndarray) or A.ndim != 2 or A.dtype != np.float64:
        raise ValueError("oracle works on 2-D float64 arrays")
    if A.shape[0] > 1 and A.strides[0] != 8:
        raise ValueError("A must be column-major")


def _cs(C, S):
    C = np.asfortranarray(C, dtype=np.float64)
    S = np.asfortranarray(S, dtype=np.float64)
    if C.shape != S.shape or C.ndim != 2:
        raise ValueError("C and S must share a 2-D shape")
    return C, S


def _lda(A):
    return max(A.strides[1] // 8 if A.shape[1] > 1 else A.shape[0], 1)


def apply_naive(A, C, S, side: str = "right", order: str = "forward", kind: str = "rotation",
                fast: bool = False, owners=None) -> None:
    """In-place semantic definition (core.py:195-205) with the side/order extensions.
    ``owners=(o0, o1)`` restricts to rows (right) / columns (left) [o0, o1)."""
    _check_A(A)
    C, S = _cs(C, S)
    m, n = A.shape
    length = m if side == "left" else n
    if C.shape[0] != length - 1:
        raise ValueError("C/S rows must equal len - 1")
    if length < 2 or m == 0 or n == 0:
        return
    o0, o1 = owners if owners is not None else (0, n if side == "left" else m)
    fn = getattr(load(), "oracle_apply_naive_f64_" + ("fast" if fast else "strict"))
    fn(A.ctypes.data, m, n, _lda(A), C.ctypes.data, S.ctypes.data, max(C.shape[0], 1), C.shape[1],
       1 if side == "left" else 0, 1 if order == "reverse" else 0, 1 if kind == "reflector" else 0, o0, o1)


def default_plan(m_r: int = DEFAULT_MR, k_r: int = DEFAULT_KR, T1=4000, T2=32000, T3=4480000, cap=4800):
    """choose_block_sizes (blocking.py:115-147) for the default CacheSpec."""
    t1_eff = T1 - math.ceil(T1 * 0.01)
    nb = (t1_eff - m_r * k_r) // (m_r + 2 * k_r)
    nbr = (nb // 8) * 8
    n_b = nbr if nbr >= k_r + 1 else nb
    kb = (T2 - m_r * n_b) // (m_r + 2 * n_b)
    k_b = (kb // k_r) * k_r
    mb = min(T3 // (n_b + k_b), cap)
    m_b = (mb // m_r) * m_r
    return dict(n_b=n_b, k_b=k_b, m_b=m_b, m_r=m_r, k_r=k_r)


def apply_blocked(A, C, S, kind: str = "rotation", fast: bool = False, threads: int = 1, plan=None) -> None:
    """The reference "kernel" tier (apply_blocked, use_kernel=True), right side forward."""
    _check_A(A)
    C, S = _cs(C, S)
    m, n = A.shape
    if m == 0:
        return
    if C.shape[0] != n - 1:
        raise ValueError("C/S rows must equal n - 1")
    p = plan or default_plan()
    fn = getattr(load(), "oracle_apply_blocked_f64_" + ("fast" if fast else "strict"))
    rc = fn(A.ctypes.data, m, n, _lda(A), C.ctypes.data, S.ctypes.data, max(C.shape[0], 1), C.shape[1],
            1 if kind == "reflector" else 0, p["n_b"], p["k_b"], p["m_b"], p["m_r"], p["k_r"], int(threads))
    if rc != 0:
        raise RuntimeError(f"oracle_apply_blocked failed ({rc})")


def partition_rows(m: int, threads: int, m_r: int):
    out = np.zeros(2 * threads, dtype=np.int64)
    load().oracle_partition_rows_strict(m, threads, m_r, out.ctypes.data)
    return [(int(out[2 * i]), int(out[2 * i + 1])) for i in range(threads)]


def numpy_apply_naive(A, C, S, side: str = "right", order: str = "forward", kind: str = "rotation") -> None:
    """Pure-numpy restatement of _naive_py (core.py:195-205) + extensions; strict
    IEEE arithmetic (numpy never contracts), vectorised across owners. Works in the
    dtype of A: float64 (the reference) or float32 (the strict fp32 oracle, with C/S
    rounded to float32)."""
    if not isinstance(A, np.ndarray) or A.ndim != 2 or A.dtype not in (np.float64, np.float32):
        raise ValueError("oracle works on 2-D float64/float32 arrays")
    if A.shape[0] > 1 and A.strides[0] != A.itemsize:
        raise ValueError("A must be column-major")
    C = np.asfortranarray(C, dtype=A.dtype)
    S = np.asfortranarray(S, dtype=A.dtype)
    X = A.T if side == "left" else A  # lines are columns of X, owners its rows
    length = X.shape[1]
    for p in range(C.shape[1]):
        js = range(length - 2, -1, -1) if order == "reverse" else range(length - 1)
        for j in js:
            c = C[j, p]
            s = S[j, p]
            xv = X[:, j].copy()
            yv = X[:, j + 1].copy()
            if kind == "reflector":
                d = c - s
                e = c + s
                w = s * (xv + yv)
                X[:, j] = w + d * xv
                X[:, j + 1] = w - e * yv
            else:
                t = c * xv + s * yv
                X[:, j + 1] = c * yv - s * xv
                X[:, j] = t


def accumulate_q(C, S, kind: str = "rotation") -> np.ndarray:
    """Explicit orthogonal Q with apply(A) = A @ Q (oracle.py:102-109)."""
    n = C.shape[0] + 1
    Q = np.eye(n, order="F")
    apply_naive(Q, C, S, kind=kind)
    return Q


def upcast_reference(A32, C32, S32, **kw) -> np.ndarray:
    """fp32 oracle: the reference arithmetic run in fp64 on the fp32-rounded inputs
    (SURVEY §8(c)); returns the fp64 result."""
    A = np.asfortranarray(A32, dtype=np.float64)
    apply_naive(A, np.asarray(C32, dtype=np.float64), np.asarray(S32, dtype=np.float64), **kw)
    return A


def wave_apply(panel, ct, st, n_waves: int, k_r: int, col0: int = 0, kind: str = "rotation") -> None:
    """Micro-kernel semantics (``_kern_generic_py``, kernels.py:81-103) on a C-contiguous
    (n_cols, m_r) panel, vectorised over the m_r rows: wave w, lane l rotates columns
    (col0 + w + k_r - 1 - l, +1) with ct/st[w * k_r + l]. Plain IEEE mul/add in the
    reference's expression order, so strict results are bit-identical."""
    P = panel
    for w in range(n_waves):
        for lane in range(k_r):
            c = ct[w * k_r + lane]
            s = st[w * k_r + lane]
            j = col0 + w + k_r - 1 - lane
            xv = P[j].copy()
            yv = P[j + 1].copy()
            if kind == "reflector":
                d = c - s
                e = c + s
                wv = s * (xv + yv)
                P[j] = wv + d * xv
                P[j + 1] = wv - e * yv
            else:
                t = c * xv + s * yv
                P[j + 1] = c * yv - s * xv
                P[j] = t


def edge_apply(panel, C, S, p0: int, k_chunk: int, triangle: str, kind: str = "rotation") -> None:
    """Startup / shutdown triangles as k_r = 1 passes (kernel_edge_apply, kernels.py:374-410)."""
    n = panel.shape[0]
    if triangle == "startup":
        for pp in range(k_chunk - 1):
            run = k_chunk - 1 - pp
            wave_apply(panel, C[0:run, p0 + pp], S[0:run, p0 + pp], run, 1, 0, kind)
    else:
        for pp in range(1, k_chunk):
            q0 = n - 1 - pp
            wave_apply(panel, C[q0:n - 1, p0 + pp], S[q0:n - 1, p0 + pp], pp, 1, q0, kind)
