"""ctypes binding of the C-ABI in ``include/rotseq_b200.h``.

The shared library ``librotseq_b200.so`` is built in-tree by
``paper_2412_01852_b200.build.build_library()`` (``__graft_entry__.build()``).
There is no fallback: if the library is missing every entry point raises,
so a CPU or eager path can never stand in for the CUDA kernels.
"""

from __future__ import annotations

import ctypes
import os
import threading

LIB_NAME = "librotseq_b200.so"
LIB_PATH = os.environ.get("RS_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

RS_OK, RS_EINVAL, RS_ECUDA, RS_ENOMEM, RS_EUNSUPPORTED = 0, 1, 2, 3, 4
STATUS_NAMES = {
    RS_OK: "RS_OK",
    RS_EINVAL: "RS_EINVAL",
    RS_ECUDA: "RS_ECUDA",
    RS_ENOMEM: "RS_ENOMEM",
    RS_EUNSUPPORTED: "RS_EUNSUPPORTED",
}
SIDE_RIGHT, SIDE_LEFT = 0, 1
ORDER_FORWARD, ORDER_REVERSE = 0, 1
KIND_ROTATION, KIND_REFLECTOR = 0, 1
DTYPE_F64, DTYPE_F32 = 0, 1
ALGO_PIPELINE, ALGO_NAIVE = 0, 1

# Every symbol include/rotseq_b200.h declares (checked by tests/test_library.py).
EXPORTS = (
    "rs_version",
    "rs_last_error",
    "rs_workspace_bytes",
    "rs_apply_f64",
    "rs_apply_f32",
    "rs_apply_algo_f64",
    "rs_apply_algo_f32",
    "rs_plan_info",
    "rs_tile_shape",
    "rs_pack_f64",
    "rs_pack_f32",
    "rs_pack_fast_f64",
    "rs_pack_fast_f32",
    "rs_apply_packed_f64",
    "rs_apply_packed_f32",
    "rs_packed_form",
    "rs_apply_host_f64",
    "rs_apply_host_f32",
    "rs_wave_apply_f64",
    "rs_wave_apply_f32",
    "rs_dmma_workspace_bytes",
    "rs_apply_dmma_f64",
    "rs_launch_count",
    "rs_debug_set_trace",
    "rs_fma_peak_tflops",
)

_lock = threading.Lock()
_lib = None


class LibraryNotBuilt(RuntimeError):
    pass


class _Partial:
    """Developer builds selected with RS_LIB_PATH may predate newer entry points: declaring
    a symbol they lack is skipped (calling it raises AttributeError)."""

    def __init__(self, lib):
        self._lib = lib

    def __getattr__(self, name):
        try:
            return getattr(self._lib, name)
        except AttributeError:
            return type("_Missing", (), {})()


def _declare(lib):
    if os.environ.get("RS_LIB_PATH"):
        lib = _Partial(lib)
    i64, i32, vp, sz = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t
    lib.rs_version.restype = i32
    lib.rs_version.argtypes = []
    lib.rs_last_error.restype = ctypes.c_char_p
    lib.rs_last_error.argtypes = []
    lib.rs_workspace_bytes.restype = sz
    lib.rs_workspace_bytes.argtypes = [i64, i64, i64, i32, i32, i32]
    apply_args = [vp, i64, i64, i64, vp, vp, i64, i64, i32, i32, i32, i32, vp, sz, vp]
    for name in ("rs_apply_f64", "rs_apply_f32"):
        fn = getattr(lib, name)
        fn.restype = i32
        fn.argtypes = apply_args
    for name in ("rs_apply_algo_f64", "rs_apply_algo_f32"):
        fn = getattr(lib, name)
        fn.restype = i32
        fn.argtypes = [i32] + apply_args
    for name in ("rs_pack_f64", "rs_pack_f32", "rs_pack_fast_f64", "rs_pack_fast_f32"):
        fn = getattr(lib, name)
        fn.restype = i32
        fn.argtypes = [vp, vp, i64, i64, i64, i64, i32, i32, i32, vp, sz, vp]
    for name in ("rs_apply_packed_f64", "rs_apply_packed_f32"):
        fn = getattr(lib, name)
        fn.restype = i32
        fn.argtypes = [vp, i64, i64, i64, i64, i32, i32, i32, i32, vp, sz, vp]
    for name in ("rs_apply_host_f64", "rs_apply_host_f32"):
        fn = getattr(lib, name)
        fn.restype = i32
        fn.argtypes = [vp, i64, i64, i64, vp, vp, i64, i64, i32, i32, i32, i32, vp]
    for name in ("rs_wave_apply_f64", "rs_wave_apply_f32"):
        fn = getattr(lib, name)
        fn.restype = i32
        fn.argtypes = [vp, i64, i64, i64, vp, vp, i64, i64, i64, i32, i32, vp]
    lib.rs_dmma_workspace_bytes.restype = sz
    lib.rs_dmma_workspace_bytes.argtypes = [i64, i64, i64]
    lib.rs_apply_dmma_f64.restype = i32
    lib.rs_apply_dmma_f64.argtypes = [vp, i64, i64, i64, vp, vp, i64, i64, i32, i32, vp, sz, vp]
    lib.rs_packed_form.restype = i32
    lib.rs_packed_form.argtypes = [vp, sz, i64, i64, i64, i32, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64), vp]
    lib.rs_plan_info.restype = i32
    lib.rs_plan_info.argtypes = [i64, i64, i64, i32, i32, i32,
                                 ctypes.POINTER(i32), ctypes.POINTER(i32), ctypes.POINTER(i64),
                                 ctypes.POINTER(i32), ctypes.POINTER(i32), ctypes.POINTER(sz)]
    lib.rs_tile_shape.restype = i32
    lib.rs_tile_shape.argtypes = [i32, i32] + [ctypes.POINTER(i32)] * 5
    lib.rs_launch_count.restype = i64
    lib.rs_launch_count.argtypes = []
    lib.rs_fma_peak_tflops.restype = i32
    lib.rs_fma_peak_tflops.argtypes = [i32, ctypes.POINTER(ctypes.c_double), vp]
    lib.rs_debug_set_trace.restype = i32
    lib.rs_debug_set_trace.argtypes = [vp]
    return lib._lib if isinstance(lib, _Partial) else lib


def load():
    """Load (once) and return the CUDA library; raise LibraryNotBuilt if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise LibraryNotBuilt(
                    f"{LIB_PATH} is missing: build the CUDA extension first "
                    "(python -c 'import __graft_entry__ as g; g.build()')"
                )
            _lib = _declare(ctypes.CDLL(LIB_PATH))
    return _lib


def last_error() -> str:
    return load().rs_last_error().decode("utf-8", "replace")


def check(status: int, what: str) -> None:
    """Map an rs_status to the reference's exception types (ValueError for bad
    arguments, core.py:41-51 / 110-117; RuntimeError otherwise)."""
    if status == RS_OK:
        return
    msg = f"{what}: {STATUS_NAMES.get(status, status)}: {last_error()}"
    if status == RS_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(msg)


def launch_count() -> int:
    return int(load().rs_launch_count())


def plan_info(m: int, n: int, k: int, side: int = SIDE_RIGHT, kind: int = KIND_ROTATION,
              dtype: int = DTYPE_F64) -> dict:
    lib = load()
    grid, nw, bw, rpt = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    units, smem = ctypes.c_int64(), ctypes.c_size_t()
    st = lib.rs_plan_info(m, n, k, side, kind, dtype, ctypes.byref(grid), ctypes.byref(nw),
                          ctypes.byref(units), ctypes.byref(bw), ctypes.byref(rpt), ctypes.byref(smem))
    check(st, "rs_plan_info")
    return dict(grid_ctas=grid.value, warps_per_cta=nw.value, units=units.value,
                band_width=bw.value, rows_per_tile=rpt.value, smem_bytes=smem.value)


def tile_shape(dtype: int = DTYPE_F64, side: int = SIDE_RIGHT) -> dict:
    """Compile-time tile shape of the pipeline kernel (no GPU needed): what
    model.choose_tile_shape must reproduce."""
    v = [ctypes.c_int() for _ in range(5)]
    check(load().rs_tile_shape(dtype, side, *[ctypes.byref(x) for x in v]), "rs_tile_shape")
    return dict(window_sweeps=v[0].value, rows_per_thread=v[1].value, ring_chunks=v[2].value,
                small_cta_warps=v[3].value, max_warps=v[4].value)


def fma_peak_tflops(dtype: int = DTYPE_F64, stream=None) -> float:
    """Live DFMA/FFMA peak of the current device (roofline denominator)."""
    out = ctypes.c_double()
    check(load().rs_fma_peak_tflops(dtype, ctypes.byref(out), stream), "rs_fma_peak_tflops")
    return out.value
