"""Drop-in entry points: apply a rotation sequence to A on a B200.

Reference operator API being replaced (same argument meaning, in-place update,
``None`` return, ``ValueError`` on bad arguments):

* ``apply_naive(A, seq, kind, fast)``              core.py:365-374
* ``apply_blocked(A, seq, plan, shape, kind,
  threads, fast, use_kernel)``                     blocking.py:420-476
* ``apply_blocked_packed`` / resident-A mode       blocking.py:479-515

``apply_cuda`` is the general form. ``A`` is either

* a host ``numpy`` array (column-major float64/float32, row-block views with
  ld > rows allowed): it is copied to the device, transformed, and copied back
  into the caller's array (the end-to-end path), or
* a CUDA ``torch.Tensor`` whose first stride is 1 (a column-major view): it is
  transformed in place on the tensor's current stream (the resident path; PyTorch
  only provides the buffer and the stream).

The arithmetic runs only in the CUDA library (``_lib``); there is no CPU fallback.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .core import (
    Order,
    RotationSequence,
    Side,
    TransformKind,
    _as_enum,
    check_apply_args,
    sequence_parts,
)

ALGOS = {"pipeline": _lib.ALGO_PIPELINE, "naive": _lib.ALGO_NAIVE}


def _torch():
    import torch  # noqa: PLC0415 - torch is plumbing, imported lazily

    return torch


def _is_tensor(x) -> bool:
    try:
        torch = _torch()
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def _np_to_device(arr: np.ndarray, dtype, device):
    """Column-major device copy of a 2-D host array (any strides)."""
    torch = _torch()
    rows, cols = arr.shape
    host = torch.from_numpy(np.asarray(arr))
    out = torch.empty_strided((rows, cols), (1, max(rows, 1)), dtype=dtype, device=device)
    out.copy_(host.to(dtype) if host.dtype != dtype else host)
    return out


def _seq_arrays(seq, dtype, device):
    """(C, S) as device tensors of `dtype` (sequence object — ours or the reference's —
    or a (C, S) pair of numpy arrays / torch tensors). Conversions and host copies are
    enqueued on the current stream of `device`."""
    C, S, _ = sequence_parts(seq)
    out = []
    for X, name in ((C, "C"), (S, "S")):
        if _is_tensor(X):
            if X.dim() != 2:
                raise ValueError(f"{name} must be 2-D")
            if X.device != device or X.dtype != dtype:
                X = X.to(device=device, dtype=dtype, non_blocking=True)
            out.append(X)
        else:
            X = np.asarray(X)
            if X.ndim != 2:
                raise ValueError(f"{name} must be 2-D")
            out.append(_np_to_device(X, dtype, device))
    if tuple(out[0].shape) != tuple(out[1].shape):
        raise ValueError(f"C and S must share a 2-D shape, got {tuple(out[0].shape)} vs {tuple(out[1].shape)}")
    return out[0], out[1]


def _seq_ncols(seq) -> int:
    return sequence_parts(seq)[2]


def _launch_stream(stream, device):
    """(launch stream, current stream). A caller-supplied stream (torch stream or raw
    cudaStream_t handle) is ordered after the current stream, on which the C/S device
    copies, casts and compaction run, so the library never reads them early."""
    torch = _torch()
    cur = torch.cuda.current_stream(device)
    if stream is None:
        return cur, cur
    if not hasattr(stream, "cuda_stream"):
        stream = torch.cuda.ExternalStream(int(stream), device=device)
    if stream.cuda_stream != cur.cuda_stream:
        stream.wait_stream(cur)
    return stream, cur


def _keep_alive(stream, cur, *tensors):
    """Tie temporaries made on `cur` to `stream` for the caching allocator."""
    if stream.cuda_stream != cur.cuda_stream:
        for X in tensors:
            X.record_stream(stream)


def apply_device(A, seq, kind=TransformKind.ROTATION, fast: bool = False, side=Side.RIGHT,
                 order=Order.FORWARD, algo: str = "pipeline", workspace=None, stream=None) -> None:
    """In-place apply on a CUDA tensor A (column-major view). Asynchronous on
    ``stream`` (default: the current torch stream of A's device)."""
    torch = _torch()
    kind = _as_enum(kind, TransformKind, "kind")
    side = _as_enum(side, Side, "side")
    order = _as_enum(order, Order, "order")
    if algo not in ALGOS:
        raise ValueError(f"unknown algorithm {algo!r}; choose from {tuple(ALGOS)}")
    if not _is_tensor(A) or not A.is_cuda:
        raise ValueError("A must be a CUDA torch.Tensor for apply_device")
    if A.dim() != 2:
        raise ValueError("A must be a 2-D tensor")
    if A.dtype not in (torch.float64, torch.float32):
        raise ValueError(f"A must have dtype float64 or float32, got {A.dtype}")
    m, n = int(A.shape[0]), int(A.shape[1])
    if m > 1 and A.stride(0) != 1:
        raise ValueError("A must be column-major (first stride 1); use A.t().contiguous().t()")
    length = m if side is Side.LEFT else n
    what = "rows" if side is Side.LEFT else "columns"
    if length < 2:
        if side is Side.LEFT:
            raise ValueError(f"matrix needs at least 2 rows for left-side application, got {m}")
        raise ValueError(f"matrix needs at least 2 columns, got {n}")
    ncols = _seq_ncols(seq)
    if ncols != length:
        raise ValueError(f"sequence acts on {ncols} {what} but matrix has {length}")
    if m == 0 or n == 0:
        return
    lda = int(A.stride(1)) if n > 1 else max(m, 1)
    C, S = _seq_arrays(seq, A.dtype, A.device)
    rows_cs, k = int(C.shape[0]), int(C.shape[1])
    if rows_cs != length - 1:
        raise ValueError(f"C/S have {rows_cs} rows, expected {length - 1}")

    def _compact(X):
        out = torch.empty_strided((rows_cs, k), (1, max(rows_cs, 1)), dtype=X.dtype, device=X.device)
        out.copy_(X)
        return out

    ldc = int(C.stride(1)) if k > 1 else max(rows_cs, 1)
    lds = int(S.stride(1)) if k > 1 else max(rows_cs, 1)
    col_major = all(X.shape[0] <= 1 or X.stride(0) == 1 for X in (C, S))
    if not col_major or ldc != lds or ldc < rows_cs:
        C, S = _compact(C), _compact(S)
        ldc = max(rows_cs, 1)
    ldcs = ldc
    lib = _lib.load()
    f64 = A.dtype == torch.float64
    dt = _lib.DTYPE_F64 if f64 else _lib.DTYPE_F32
    side_i = _lib.SIDE_LEFT if side is Side.LEFT else _lib.SIDE_RIGHT
    kind_i = _lib.KIND_REFLECTOR if kind is TransformKind.REFLECTOR else _lib.KIND_ROTATION
    order_i = _lib.ORDER_REVERSE if order is Order.REVERSE else _lib.ORDER_FORWARD
    ws_ptr, ws_bytes = None, 0
    if workspace is not None:
        need = lib.rs_workspace_bytes(m, n, k, side_i, kind_i, dt)
        if workspace.numel() * workspace.element_size() < need:
            raise ValueError(f"workspace too small: need {need} bytes")
        ws_ptr, ws_bytes = workspace.data_ptr(), workspace.numel() * workspace.element_size()
    with torch.cuda.device(A.device):
        lstream, cur = _launch_stream(stream, A.device)
        fn = lib.rs_apply_algo_f64 if f64 else lib.rs_apply_algo_f32
        st = fn(ALGOS[algo], A.data_ptr(), m, n, lda, C.data_ptr(), S.data_ptr(), ldcs, k,
                side_i, order_i, kind_i, 0 if fast else 1, ws_ptr, ws_bytes, lstream.cuda_stream)
        # C/S may be temporaries from torch's caching allocator: tie them to the launch stream
        _keep_alive(lstream, cur, C, S)
    _lib.check(st, "rs_apply")


def _host_cs(seq, np_dtype, length):
    """(C, S) as host column-major arrays of the working dtype (copies only if needed)."""
    C, S, _ = sequence_parts(seq)
    out = []
    for X, name in ((C, "C"), (S, "S")):
        if _is_tensor(X):
            if X.is_cuda:
                raise ValueError(f"{name} is a CUDA tensor but A is in host memory")
            X = X.numpy()
        X = np.asarray(X)
        if X.ndim != 2:
            raise ValueError(f"{name} must be 2-D")
        out.append(np.asfortranarray(X, dtype=np_dtype))
    if out[0].shape != out[1].shape:
        raise ValueError(f"C and S must share a 2-D shape, got {out[0].shape} vs {out[1].shape}")
    if out[0].shape[0] != length - 1:
        raise ValueError(f"C/S have {out[0].shape[0]} rows, expected {length - 1}")
    return out[0], out[1]


def apply_host(A, seq, kind=TransformKind.ROTATION, fast: bool = False, side=Side.RIGHT,
               order=Order.FORWARD, device=None) -> None:
    """In-place apply on a host matrix (numpy array or CPU torch tensor, column-major)
    through ``rs_apply_host_*``: C/S are copied and packed, then A streams to the GPU
    and back in wave-column chunks overlapped with the kernel. Synchronous. Pinned
    memory (``torch.empty(..., pin_memory=True)``) gives full copy bandwidth."""
    torch = _torch()
    kind = _as_enum(kind, TransformKind, "kind")
    side = _as_enum(side, Side, "side")
    order = _as_enum(order, Order, "order")
    if _is_tensor(A):
        if A.is_cuda:
            raise ValueError("apply_host needs a host matrix; use apply_device for CUDA tensors")
        if A.dim() != 2 or A.dtype not in (torch.float64, torch.float32):
            raise ValueError("A must be a 2-D float64/float32 tensor")
        if A.shape[0] > 1 and A.stride(0) != 1:
            raise ValueError("A must be column-major (first stride 1)")
        m, n = int(A.shape[0]), int(A.shape[1])
        lda = int(A.stride(1)) if n > 1 else max(m, 1)
        np_dtype = np.float64 if A.dtype == torch.float64 else np.float32
        ptr = A.data_ptr()
    else:
        check_apply_args(A, seq, side, dtypes=(np.float64, np.float32))
        m, n = A.shape
        lda = A.strides[1] // A.itemsize if n > 1 else max(m, 1)
        np_dtype = A.dtype.type
        ptr = A.ctypes.data
    length = m if side is Side.LEFT else n
    if length < 2:
        if side is Side.LEFT:
            raise ValueError(f"matrix needs at least 2 rows for left-side application, got {m}")
        raise ValueError(f"matrix needs at least 2 columns, got {n}")
    ncols = _seq_ncols(seq)
    if ncols != length:
        what = "rows" if side is Side.LEFT else "columns"
        raise ValueError(f"sequence acts on {ncols} {what} but matrix has {length}")
    if m == 0 or n == 0:
        return
    C, S = _host_cs(seq, np_dtype, length)
    k = C.shape[1]
    lib = _lib.load()
    f64 = np_dtype == np.float64
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev)
        fn = lib.rs_apply_host_f64 if f64 else lib.rs_apply_host_f32
        st = fn(ptr, m, n, lda, C.ctypes.data, S.ctypes.data, max(C.shape[0], 1), k,
                _lib.SIDE_LEFT if side is Side.LEFT else _lib.SIDE_RIGHT,
                _lib.ORDER_REVERSE if order is Order.REVERSE else _lib.ORDER_FORWARD,
                _lib.KIND_REFLECTOR if kind is TransformKind.REFLECTOR else _lib.KIND_ROTATION,
                0 if fast else 1, stream.cuda_stream)
    _lib.check(st, "rs_apply_host")


def workspace_bytes(m: int, n: int, k: int, side=Side.RIGHT, kind=TransformKind.ROTATION,
                    dtype=np.float64) -> int:
    side = _as_enum(side, Side, "side")
    kind = _as_enum(kind, TransformKind, "kind")
    lib = _lib.load()
    dt = _lib.DTYPE_F64 if np.dtype(dtype) == np.float64 else _lib.DTYPE_F32
    return int(lib.rs_workspace_bytes(m, n, k, _lib.SIDE_LEFT if side is Side.LEFT else _lib.SIDE_RIGHT,
                                      _lib.KIND_REFLECTOR if kind is TransformKind.REFLECTOR else _lib.KIND_ROTATION,
                                      dt))


def apply_cuda(A, seq, kind=TransformKind.ROTATION, fast: bool = False, side=Side.RIGHT,
               order=Order.FORWARD, algo: str = "pipeline", device=None, workspace=None) -> None:
    """Apply the sequence to A in place on the GPU; returns None.

    Host numpy input: validated like the reference (``_check_apply_args``,
    core.py:110-117), copied to ``device`` (default cuda:current), transformed,
    copied back, synchronised. Device tensor input: see ``apply_device``.
    """
    torch = _torch()
    if _is_tensor(A) and A.is_cuda:
        apply_device(A, seq, kind, fast, side, order, algo, workspace)
        return
    if algo == "pipeline":
        # host matrix: the streaming host-buffer C-ABI (copies overlap the kernel)
        apply_host(A, seq, kind, fast, side, order, device)
        return
    if _is_tensor(A):
        # host torch tensor (ideally pinned): async H2D, apply, async D2H, synchronise
        if A.dim() != 2 or A.dtype not in (torch.float64, torch.float32):
            raise ValueError("A must be a 2-D float64/float32 tensor")
        if A.shape[0] > 1 and A.stride(0) != 1:
            raise ValueError("A must be column-major (first stride 1)")
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        m, n = A.shape
        dA = torch.empty_strided((m, n), (1, max(m, 1)), dtype=A.dtype, device=dev)
        dA.copy_(A, non_blocking=True)
        apply_device(dA, seq, kind, fast, side, order, algo, workspace)
        A.copy_(dA, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
        return
    kind = _as_enum(kind, TransformKind, "kind")
    side = _as_enum(side, Side, "side")
    order = _as_enum(order, Order, "order")
    check_apply_args(A, seq, side, dtypes=(np.float64, np.float32))
    if A.shape[0] == 0 or A.shape[1] == 0:
        return
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    tdt = torch.float64 if A.dtype == np.float64 else torch.float32
    dA = _np_to_device(A, tdt, dev)
    apply_device(dA, seq, kind, fast, side, order, algo, workspace)
    torch.from_numpy(A).copy_(dA.cpu())


def apply_naive(A, seq: RotationSequence, kind=TransformKind.ROTATION, fast: bool = False) -> None:
    """Reference signature (core.py:365-374), executed by the B200 pipeline.

    ``seq`` may be this package's ``RotationSequence``, the reference's own
    ``rotseq.RotationSequence`` or a ``(C, S)`` pair; ``kind`` may be either package's
    ``TransformKind`` or its string value. Result is bit-identical to the reference's
    strict ``apply_naive`` when ``fast`` is False (every variant in the reference is,
    SPEC criterion 1)."""
    apply_cuda(A, seq, kind=kind, fast=fast)


def apply_blocked(A, seq: RotationSequence, plan=None, shape=None, kind=TransformKind.ROTATION,
                  threads: int = 1, fast: bool = False, use_kernel: bool = True) -> None:
    """Reference signature (blocking.py:420-429). ``plan``/``shape``/``threads``
    are CPU cache and thread knobs; the GPU tiling is chosen by the library, so
    they are validated for sign only and otherwise ignored."""
    if threads < 1:
        raise ValueError(f"threads must be >= 1, got {threads}")
    apply_cuda(A, seq, kind=kind, fast=fast)


class PackedSequence:
    """Coefficients packed once into device memory for repeated application.

    GPU counterpart of the reference's prepacked path (``apply_blocked_packed``,
    blocking.py:479-515; the paper's rs_kernel_v2): ``pack`` runs the
    repack kernel into a persistent workspace, ``apply`` runs only the pipeline kernel
    on a device-resident A. Shape, side, order and kind are fixed at construction.
    ``fast_only=True`` packs for fast-mode application only (``rs_pack_fast_*``: the
    standard records are written only when the scaled form is out of range), which
    makes every re-pack cheaper; ``apply(fast=False)`` is then refused.
    """

    def __init__(self, seq, shape, kind=TransformKind.ROTATION, side=Side.RIGHT, order=Order.FORWARD,
                 dtype=None, device=None, stream=None, fast_only=False):
        torch = _torch()
        self.fast_only = bool(fast_only)
        self.kind = _as_enum(kind, TransformKind, "kind")
        self.side = _as_enum(side, Side, "side")
        self.order = _as_enum(order, Order, "order")
        self.m, self.n = int(shape[0]), int(shape[1])
        self.length = self.m if self.side is Side.LEFT else self.n
        ncols = _seq_ncols(seq)
        what = "rows" if self.side is Side.LEFT else "columns"
        if self.length < 2:
            raise ValueError(f"matrix needs at least 2 {what}")
        if ncols != self.length:
            raise ValueError(f"sequence acts on {ncols} {what} but matrix has {self.length}")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        if dtype is None:
            dtype = torch.float64
        self.dtype = dtype
        self.f64 = dtype == torch.float64
        lib = _lib.load()
        self._side = _lib.SIDE_LEFT if self.side is Side.LEFT else _lib.SIDE_RIGHT
        self._kind = _lib.KIND_REFLECTOR if self.kind is TransformKind.REFLECTOR else _lib.KIND_ROTATION
        self._order = _lib.ORDER_REVERSE if self.order is Order.REVERSE else _lib.ORDER_FORWARD
        C, S = _seq_arrays(seq, dtype, self.device)
        self.k = int(C.shape[1])
        nbytes = lib.rs_workspace_bytes(self.m, self.n, self.k, self._side, self._kind,
                                        _lib.DTYPE_F64 if self.f64 else _lib.DTYPE_F32)
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self.pack((C, S), stream)


    def pack(self, seq, stream=None) -> None:
        """(Re)pack new coefficients of the same shape into the workspace."""
        torch = _torch()
        C, S = _seq_arrays(seq, self.dtype, self.device)
        if tuple(C.shape) != (self.length - 1, self.k):
            raise ValueError(f"C/S must be {(self.length - 1, self.k)}, got {tuple(C.shape)}")
        if not all(X.shape[0] <= 1 or X.stride(0) == 1 for X in (C, S)) or C.stride(1) != S.stride(1):
            C, S = C.t().contiguous().t(), S.t().contiguous().t()
        ldcs = int(C.stride(1)) if self.k > 1 else max(self.length - 1, 1)
        lib = _lib.load()
        if self.fast_only:
            fn = lib.rs_pack_fast_f64 if self.f64 else lib.rs_pack_fast_f32
        else:
            fn = lib.rs_pack_f64 if self.f64 else lib.rs_pack_f32
        with torch.cuda.device(self.device):
            lstream, cur = _launch_stream(stream, self.device)
            st = fn(C.data_ptr(), S.data_ptr(), ldcs, self.m, self.n, self.k, self._side, self._order, self._kind,
                    self.workspace.data_ptr(), self.workspace.numel(), lstream.cuda_stream)
            _keep_alive(lstream, cur, C, S, self.workspace)
        _lib.check(st, "rs_pack")

    def form(self, stream=None):
        """(scaled_units, total_units): how many units a fast-mode ``apply`` runs in the
        scaled (fast Givens) form; the others use the standard fast form because their
        coefficients leave the scaled form's safe range. Synchronous (``rs_packed_form``)."""
        import ctypes  # noqa: PLC0415

        torch = _torch()
        lib = _lib.load()
        scaled, total = ctypes.c_int64(), ctypes.c_int64()
        with torch.cuda.device(self.device):
            lstream, _ = _launch_stream(stream, self.device)
            st = lib.rs_packed_form(self.workspace.data_ptr(), self.workspace.numel(), self.m, self.n, self.k,
                                    self._side, self._kind, _lib.DTYPE_F64 if self.f64 else _lib.DTYPE_F32,
                                    ctypes.byref(scaled), ctypes.byref(total), lstream.cuda_stream)
        _lib.check(st, "rs_packed_form")
        return int(scaled.value), int(total.value)

    def apply(self, A, fast: bool = False, stream=None) -> None:
        """Apply the packed sequence to the CUDA tensor A (column-major) in place."""
        torch = _torch()
        if not _is_tensor(A) or not A.is_cuda or A.dtype != self.dtype:
            raise ValueError("A must be a CUDA tensor of the packed dtype")
        if tuple(A.shape) != (self.m, self.n):
            raise ValueError(f"A must have shape {(self.m, self.n)}, got {tuple(A.shape)}")
        if self.m > 1 and A.stride(0) != 1:
            raise ValueError("A must be column-major (first stride 1)")
        if self.fast_only and not fast:
            raise ValueError("this PackedSequence was packed fast_only; apply it with fast=True")
        lda = int(A.stride(1)) if self.n > 1 else max(self.m, 1)
        lib = _lib.load()
        fn = lib.rs_apply_packed_f64 if self.f64 else lib.rs_apply_packed_f32
        with torch.cuda.device(self.device):
            lstream, cur = _launch_stream(stream, self.device)
            st = fn(A.data_ptr(), self.m, self.n, lda, self.k, self._side, self._order, self._kind,
                    0 if fast else 1, self.workspace.data_ptr(), self.workspace.numel(), lstream.cuda_stream)
            _keep_alive(lstream, cur, self.workspace)
        _lib.check(st, "rs_apply_packed")


def apply_dmma(A, seq, kind=TransformKind.ROTATION, order=Order.FORWARD, workspace=None, stream=None) -> None:
    """The FP64 tensor-core (DMMA) accumulate-and-apply variant (``rs_apply_dmma_f64``;
    the paper's rs_gemm): right side, fp64, fast-mode accuracy. ``A`` is a
    column-major CUDA float64 tensor (updated in place on ``stream``) or a host array
    (copied to the device and back)."""
    torch = _torch()
    kind = _as_enum(kind, TransformKind, "kind")
    order = _as_enum(order, Order, "order")
    if not (_is_tensor(A) and A.is_cuda):
        check_apply_args(A, seq, Side.RIGHT)
        dev = torch.device("cuda", torch.cuda.current_device())
        dA = _np_to_device(np.asarray(A), torch.float64, dev)
        apply_dmma(dA, seq, kind, order, workspace, stream)
        if isinstance(A, np.ndarray):
            A[...] = dA.cpu().numpy()
        else:
            A.copy_(dA.cpu())
        return
    if A.dim() != 2 or A.dtype != torch.float64:
        raise ValueError("the DMMA variant needs a 2-D float64 matrix")
    m, n = int(A.shape[0]), int(A.shape[1])
    if m > 1 and A.stride(0) != 1:
        raise ValueError("A must be column-major (first stride 1)")
    if n < 2:
        raise ValueError(f"matrix needs at least 2 columns, got {n}")
    ncols = _seq_ncols(seq)
    if ncols != n:
        raise ValueError(f"sequence acts on {ncols} columns but matrix has {n}")
    if m == 0:
        return
    C, S = _seq_arrays(seq, torch.float64, A.device)
    rows_cs, k = int(C.shape[0]), int(C.shape[1])
    if not all(X.shape[0] <= 1 or X.stride(0) == 1 for X in (C, S)) or C.stride(1) != S.stride(1):
        C, S = C.t().contiguous().t(), S.t().contiguous().t()
    ldcs = int(C.stride(1)) if k > 1 else max(rows_cs, 1)
    lda = int(A.stride(1)) if n > 1 else max(m, 1)
    lib = _lib.load()
    ws_ptr, ws_bytes = None, 0
    if workspace is not None:
        ws_ptr, ws_bytes = workspace.data_ptr(), workspace.numel() * workspace.element_size()
    with torch.cuda.device(A.device):
        lstream, cur = _launch_stream(stream, A.device)
        st = lib.rs_apply_dmma_f64(A.data_ptr(), m, n, lda, C.data_ptr(), S.data_ptr(), ldcs, k,
                                   _lib.ORDER_REVERSE if order is Order.REVERSE else _lib.ORDER_FORWARD,
                                   _lib.KIND_REFLECTOR if kind is TransformKind.REFLECTOR else _lib.KIND_ROTATION,
                                   ws_ptr, ws_bytes, lstream.cuda_stream)
        _keep_alive(lstream, cur, C, S)
    _lib.check(st, "rs_apply_dmma")


def dmma_workspace_bytes(m: int, n: int, k: int) -> int:
    return int(_lib.load().rs_dmma_workspace_bytes(m, n, k))
