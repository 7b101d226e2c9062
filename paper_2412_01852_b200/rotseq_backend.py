"""Register the B200 path as an algorithm of the reference package ``rotseq``.

This is the hookup INTEGRATION.md §2 describes, as executable code: the reference
dispatches every algorithm by name through ``rotseq.verification.run_variant``
(verification.py:50-85, registry ``ALGORITHMS`` verification.py:42, CLI ``--algo``
choices cli.py:346). ``register(rotseq)`` adds ``"cuda"`` to that registry at run time,
without editing the reference:

    import rotseq
    from paper_2412_01852_b200 import rotseq_backend
    rotseq_backend.register(rotseq)
    rotseq.verification.run_variant("cuda", A, seq, rotseq.TransformKind.ROTATION, fast=True)

The new entry takes the reference's own objects (``rotseq.RotationSequence``,
``rotseq.TransformKind``) and host ``numpy`` matrices, applies the sequence on the GPU
through the C-ABI (``apply_cuda`` → ``rs_apply_host_*``: copies streamed in and out around
the kernel), and then runs the reference's own fault hook (``_maybe_perturb``), exactly
as the reference treats its kernel tiers (verification.py:76, 83).
"""

from __future__ import annotations

import importlib

from .apply import apply_cuda

ALGO_NAME = "cuda"


def apply_host(A, seq, kind="rotation", fast: bool = False) -> None:
    """The reference calling convention (``apply_naive(A, seq, kind, fast)``,
    core.py:365-374) on the B200: A host column-major float64, modified in place."""
    apply_cuda(A, seq, kind=kind, fast=fast)


def register(rotseq=None, name: str = ALGO_NAME):
    """Add ``name`` to the reference's dispatcher (idempotent). ``rotseq`` is the
    imported reference package (default: ``import rotseq``). Returns the patched
    ``rotseq.verification`` module."""
    if rotseq is None:
        rotseq = importlib.import_module("rotseq")
    ver = importlib.import_module(rotseq.__name__ + ".verification")
    if getattr(ver.run_variant, "_b200_algo", None) == name:
        return ver
    base = ver.run_variant

    def run_variant(algo, A, seq, kind=ver.TransformKind.ROTATION, fast=False, plan=None, shape=None,
                    n_r=2, k_r=2, threads=1):
        if algo == name:
            if threads < 1:
                raise ValueError(f"threads must be >= 1, got {threads}")
            apply_host(A, seq, kind, fast)
            ver._maybe_perturb(A)
            return None
        return base(algo, A, seq, kind, fast, plan, shape, n_r, k_r, threads)

    run_variant._b200_algo = name
    run_variant.__doc__ = base.__doc__
    ver.run_variant = run_variant
    if name not in ver.ALGORITHMS:
        ver.ALGORITHMS = tuple(ver.ALGORITHMS) + (name,)
    # modules that imported the names (package root, CLI) see the new entry too
    for modname in (rotseq.__name__, rotseq.__name__ + ".cli"):
        try:
            mod = importlib.import_module(modname)
        except ImportError:  # pragma: no cover - CLI absent
            continue
        if getattr(mod, "run_variant", None) is base:
            mod.run_variant = run_variant
        if hasattr(mod, "ALGORITHMS"):
            mod.ALGORITHMS = ver.ALGORITHMS
    return ver
