"""Micro-kernel API on packed panels (mirror of rotseq.kernels, kernels.py:34-422).

The reference exposes its register-reuse micro-kernels as a public API that its tests
exercise standalone (the blocked driver inlines its own loop and never calls them,
SURVEY §2 note):

* ``KernelShape(m_r, k_r, vector_width, mode)``    kernels.py:34-64
* ``PanelView(base, n_cols, m_r)``                 kernels.py:67-78
* ``kernel_wave_apply(panel, C_tile, S_tile, n_waves, shape, kind, col0)``
                                                    kernels.py:335-371
* ``kernel_edge_apply(panel, C, S, p0, k_chunk, triangle, shape, kind)``
                                                    kernels.py:374-410
* ``edge_traversal(n, k_chunk, triangle)``          kernels.py:413-422

A panel is a C-contiguous ``(n_cols, m_r)`` float64 array — column j holds m_r
contiguous rows. Wave w, lane l rotates columns (col0 + w + k_r - 1 - l, +1) with the
wave-major tile entries ``tile[w * k_r + l]``. Here the waves run on the GPU through
``rs_wave_apply_*`` (one thread per panel row, the (k_r+1)-column window in registers):
a host ``numpy`` panel is copied to the device and back, a CUDA ``torch.Tensor`` panel
is updated in place on its current stream. Strict mode (``shape.mode == "strict"``)
is bit-identical to the reference; fast mode uses FMAs. There is no CPU path.

The reference's fixed-shape specialisations ((16,2), (12,3), (8,5), (48,1)) are
bit-identical to its generic kernel, so ``force_generic`` is accepted and has no
effect here (one kernel template, instantiated per k_r <= 8).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import TransformKind, _as_enum


@dataclass(frozen=True)
class KernelShape:
    """Micro-kernel tile: m_r rows per panel, k_r transforms per wave (kernels.py:34-64).
    ``vector_width`` is informational (the reference uses it for a CPU register-budget
    warning, which does not apply to a GPU thread)."""

    m_r: int
    k_r: int
    vector_width: int = 4
    mode: str = "strict"

    def __post_init__(self):
        if self.m_r < 1 or self.k_r < 1:
            raise ValueError(f"kernel shape must be positive, got {self.m_r}x{self.k_r}")
        if self.mode not in ("strict", "fast"):
            raise ValueError(f"mode must be 'strict' or 'fast', got {self.mode!r}")

    @property
    def fast(self) -> bool:
        return self.mode == "fast"


@dataclass(frozen=True)
class PanelView:
    """Column j of the panel occupies m_r contiguous values at ``base + j * m_r``
    (kernels.py:67-78)."""

    base: int
    n_cols: int
    m_r: int

    def as_array(self, buffer):
        end = self.base + self.n_cols * self.m_r
        return buffer[self.base:end].reshape(self.n_cols, self.m_r)


def _torch():
    import torch  # noqa: PLC0415 - plumbing only

    return torch


def _is_cuda_tensor(x) -> bool:
    try:
        torch = _torch()
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor) and x.is_cuda


def _check_panel(panel) -> None:
    """kernels.py:325-332: a C-contiguous (n_cols, m_r) float64 array (or such a CUDA
    tensor, float64/float32)."""
    if _is_cuda_tensor(panel):
        torch = _torch()
        if panel.dim() != 2 or panel.dtype not in (torch.float64, torch.float32) or not panel.is_contiguous():
            raise ValueError("panel must be a C-contiguous (n_cols, m_r) float64 array")
        return
    if (not isinstance(panel, np.ndarray) or panel.ndim != 2 or panel.dtype != np.float64
            or not panel.flags.c_contiguous):
        raise ValueError("panel must be a C-contiguous (n_cols, m_r) float64 array")


class _DevicePanel:
    """The panel on the device for the duration of one API call: a CUDA tensor as is, a
    host array copied in (and back on ``finish``)."""

    def __init__(self, panel):
        torch = _torch()
        self.host = None if _is_cuda_tensor(panel) else panel
        if self.host is None:
            self.dev = panel
        else:
            self.dev = torch.from_numpy(panel).to(torch.device("cuda", torch.cuda.current_device()))
        self.f64 = self.dev.dtype == torch.float64

    def tiles(self, ct, st):
        torch = _torch()
        dt = self.dev.dtype
        out = []
        for X in (ct, st):
            if isinstance(X, torch.Tensor):
                X = X.to(device=self.dev.device, dtype=dt).contiguous()
            else:
                X = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float64)).to(self.dev.device, dt)
            out.append(X)
        return out

    def run(self, ct, st, n_waves, k_r, col0, kind, strict):
        torch = _torch()
        lib = _lib.load()
        n_cols, m_r = int(self.dev.shape[0]), int(self.dev.shape[1])
        fn = lib.rs_wave_apply_f64 if self.f64 else lib.rs_wave_apply_f32
        with torch.cuda.device(self.dev.device):
            stream = torch.cuda.current_stream(self.dev.device)
            st_ = fn(self.dev.data_ptr(), m_r, n_cols, max(m_r, 1), ct.data_ptr(), st.data_ptr(), n_waves, k_r, col0,
                     _lib.KIND_REFLECTOR if kind is TransformKind.REFLECTOR else _lib.KIND_ROTATION,
                     0 if not strict else 1, stream.cuda_stream)
        _lib.check(st_, "rs_wave_apply")

    def finish(self):
        if self.host is not None:
            self.host[...] = self.dev.cpu().numpy()


def _kind(kind):
    return TransformKind.ROTATION if kind is None else _as_enum(kind, TransformKind, "kind")


def kernel_wave_apply(panel, C_tile, S_tile, n_waves: int, shape: KernelShape, kind=None, col0: int = 0,
                      force_generic: bool = False) -> None:
    """Apply n_waves waves of k_r transforms to a packed panel (kernels.py:335-371).

    ``C_tile``/``S_tile`` are wave-major: one (c, s) per (wave, lane)."""
    del force_generic  # one kernel; the reference's specialisations are bit-identical to its generic one
    _check_panel(panel)
    if panel.shape[1] != shape.m_r:
        raise ValueError(f"panel holds {panel.shape[1]} rows, shape wants {shape.m_r}")
    if panel.shape[0] - col0 < n_waves + shape.k_r:
        raise ValueError(
            f"panel has {panel.shape[0] - col0} usable columns, need "
            f"{n_waves + shape.k_r} for {n_waves} waves of {shape.k_r}"
        )
    size = (lambda X: X.numel()) if _is_cuda_tensor(C_tile) else (lambda X: np.asarray(X).size)
    if size(C_tile) < n_waves * shape.k_r or size(S_tile) < n_waves * shape.k_r:
        raise ValueError("coefficient tiles shorter than n_waves * k_r")
    kind = _kind(kind)
    dp = _DevicePanel(panel)
    ct, st = dp.tiles(C_tile, S_tile)
    dp.run(ct.reshape(-1), st.reshape(-1), n_waves, shape.k_r, col0, kind, not shape.fast)
    dp.finish()


def kernel_edge_apply(panel, C, S, p0: int, k_chunk: int, triangle: str, shape: KernelShape, kind=None) -> None:
    """A chunk's startup or shutdown triangle as k_r = 1 waves (kernels.py:374-410): the
    startup triangle runs, for each sequence offset pp, the rotations [0, k_chunk-2-pp];
    the shutdown triangle runs [n-1-pp, n-2]."""
    _check_panel(panel)
    if triangle not in ("startup", "shutdown"):
        raise ValueError(f"triangle must be 'startup' or 'shutdown', got {triangle!r}")
    kind = _kind(kind)
    n = int(panel.shape[0])
    dp = _DevicePanel(panel)
    Cd, Sd = dp.tiles(C, S)  # (n-1) x k on the device, row-major
    if triangle == "startup":
        for pp in range(k_chunk - 1):
            run = k_chunk - 1 - pp
            dp.run(Cd[0:run, p0 + pp].contiguous(), Sd[0:run, p0 + pp].contiguous(), run, 1, 0, kind,
                   not shape.fast)
    else:
        for pp in range(1, k_chunk):
            q0 = n - 1 - pp
            dp.run(Cd[q0:n - 1, p0 + pp].contiguous(), Sd[q0:n - 1, p0 + pp].contiguous(), pp, 1, q0, kind,
                   not shape.fast)
    dp.finish()


def edge_traversal(n: int, k_chunk: int, triangle: str):
    """(q, pp) order of kernel_edge_apply, pp relative to the chunk (kernels.py:413-422)."""
    if triangle == "startup":
        for pp in range(k_chunk - 1):
            for q in range(k_chunk - 1 - pp):
                yield q, pp
    else:
        for pp in range(1, k_chunk):
            for q in range(n - 1 - pp, n - 1):
                yield q, pp
