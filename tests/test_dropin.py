"""The drop-in boundary takes the reference's own objects (CPU, no GPU needed).

The reference package ``rotseq`` is imported from /root/reference (build container
only; skipped elsewhere). Its ``RotationSequence`` and ``TransformKind`` are passed
through this build's ``apply_naive`` / ``apply_blocked`` / ``run_variant`` and through
the reference's own ``run_variant`` after ``rotseq_backend.register``; the last hop —
the ctypes call into ``librotseq_b200.so`` — is replaced by a recorder, so the test
checks exactly what would reach the C-ABI (pointers, sizes, kind, strict flag).
Reference: core.py:29-38, 54-91, 365-374; blocking.py:420-429; verification.py:50-85.
"""

from __future__ import annotations

import contextlib
import ctypes
import os
import sys
import types

import numpy as np
import pytest

REF_SRC = "/root/reference/pkg/src"


@pytest.fixture(scope="module")
def rotseq():
    if not os.path.isdir(os.path.join(REF_SRC, "rotseq")):
        pytest.skip("reference package not present (GPU box)")
    pytest.importorskip("numba")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import rotseq as mod
    import rotseq.cli  # noqa: F401 - submodules as attributes
    import rotseq.verification  # noqa: F401

    return mod


class _Recorder:
    """Stands in for the loaded CUDA library: records rs_apply_host_* calls."""

    def __init__(self):
        self.calls = []

    def _host(self, name):
        def fn(ptr, m, n, lda, cptr, sptr, ldcs, k, side, order, kind, strict, stream):
            C = np.ctypeslib.as_array(ctypes.cast(cptr, ctypes.POINTER(ctypes.c_double)), shape=(k, ldcs)).T.copy()
            S = np.ctypeslib.as_array(ctypes.cast(sptr, ctypes.POINTER(ctypes.c_double)), shape=(k, ldcs)).T.copy()
            self.calls.append(dict(fn=name, ptr=ptr, m=m, n=n, lda=lda, C=C, S=S, k=k, side=side, order=order,
                                   kind=kind, strict=strict))
            return 0
        return fn

    def __getattr__(self, name):
        if name.startswith("rs_apply_host_"):
            return self._host(name)
        raise AttributeError(name)


@pytest.fixture()
def recorder(monkeypatch):
    import torch

    from paper_2412_01852_b200 import _lib

    rec = _Recorder()
    monkeypatch.setattr(_lib, "load", lambda: rec)
    monkeypatch.setattr(torch.cuda, "current_device", lambda: 0)
    monkeypatch.setattr(torch.cuda, "device", lambda dev: contextlib.nullcontext())
    monkeypatch.setattr(torch.cuda, "current_stream", lambda dev=None: types.SimpleNamespace(cuda_stream=0))
    return rec


def _check_call(call, A, seq, kind, strict):
    assert call["fn"] == "rs_apply_host_f64"
    assert call["ptr"] == A.ctypes.data  # in place: the caller's buffer
    assert (call["m"], call["n"], call["lda"], call["k"]) == (A.shape[0], A.shape[1], A.shape[0], seq.k)
    assert call["kind"] == kind and call["strict"] == strict and call["side"] == 0 and call["order"] == 0
    np.testing.assert_array_equal(call["C"], seq.C)
    np.testing.assert_array_equal(call["S"], seq.S)


def test_reference_objects_reach_the_c_abi(rotseq, recorder):
    from paper_2412_01852_b200 import apply_blocked, apply_naive, run_variant

    A, seq = rotseq.verification.make_inputs(37, 29, 5, 3)
    assert type(seq).__module__.startswith("rotseq")
    apply_naive(A, seq, rotseq.TransformKind.REFLECTOR)
    _check_call(recorder.calls[-1], A, seq, kind=1, strict=1)
    apply_blocked(A, seq, rotseq.verification.default_plan(), rotseq.verification.default_shape(),
                  kind=rotseq.TransformKind.ROTATION, threads=4, fast=True)
    _check_call(recorder.calls[-1], A, seq, kind=0, strict=0)
    run_variant("cuda", A, seq, rotseq.TransformKind.REFLECTOR, False, rotseq.verification.default_plan())
    _check_call(recorder.calls[-1], A, seq, kind=1, strict=1)
    assert len(recorder.calls) == 3


def test_reference_validation_messages(rotseq, recorder):
    """Errors raise before any GPU work, with the reference's message substrings."""
    from paper_2412_01852_b200 import apply_naive

    A, seq = rotseq.verification.make_inputs(10, 8, 2, 0)
    with pytest.raises(ValueError, match="acts on"):
        apply_naive(np.asfortranarray(A[:, :7]), seq)
    with pytest.raises(ValueError, match="column-major"):
        apply_naive(np.ascontiguousarray(A), seq)
    with pytest.raises(ValueError, match="kind"):
        apply_naive(A, seq, "householder")
    assert recorder.calls == []


def test_register_into_reference_dispatcher(rotseq, recorder):
    """INTEGRATION.md §2 as code: the reference's run_variant gains "cuda"."""
    from paper_2412_01852_b200 import rotseq_backend

    ver = rotseq_backend.register(rotseq)
    assert "cuda" in ver.ALGORITHMS and "cuda" in rotseq.verification.ALGORITHMS
    A, seq = rotseq.verification.make_inputs(20, 12, 3, 1)
    rotseq.verification.run_variant("cuda", A, seq, rotseq.TransformKind.ROTATION, fast=True, threads=2)
    _check_call(recorder.calls[-1], A, seq, kind=0, strict=0)
    # the reference's own algorithms still run through the reference
    B = A.copy(order="F")
    rotseq.verification.run_variant("naive", B, seq)
    assert len(recorder.calls) == 1
    assert rotseq_backend.register(rotseq) is ver  # idempotent
    # the reference's fault hook applies to the new kernel path, as to its own kernels
    os.environ[ver.FAULT_ENV] = "1"
    try:
        C0 = A.copy(order="F")
        rotseq.verification.run_variant("cuda", C0, seq)
        assert C0.flat[0] == np.nextafter(A.flat[0], np.inf)
    finally:
        os.environ.pop(ver.FAULT_ENV, None)


def test_duck_typed_sequence_and_enum(recorder):
    """Any object with .C/.S (and optionally .n_cols) and any enum with a matching .value."""
    import enum

    from paper_2412_01852_b200 import apply_naive, generate_sequence, make_inputs

    class Kind(enum.Enum):
        ROTATION = "rotation"
        REFLECTOR = "reflector"

    A, seq = make_inputs(16, 9, 4, 0)
    duck = types.SimpleNamespace(C=seq.C, S=seq.S, n_cols=9, k=4)
    apply_naive(A, duck, Kind.REFLECTOR)
    _check_call(recorder.calls[-1], A, seq, kind=1, strict=1)
    no_ncols = types.SimpleNamespace(C=seq.C, S=seq.S, k=4)
    apply_naive(A, no_ncols)
    _check_call(recorder.calls[-1], A, seq, kind=0, strict=1)
    with pytest.raises(ValueError, match="acts on"):
        apply_naive(A, generate_sequence(8, 4, 1))
