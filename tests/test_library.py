"""The C-ABI library: it builds for sm_100a, loads on a CPU-only host, exports every
symbol include/rotseq_b200.h declares, and validates arguments before touching the
GPU (no compute calls here)."""

from __future__ import annotations

import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT
from paper_2412_01852_b200 import _lib

HEADER = os.path.join(ROOT, "include", "rotseq_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rs_[a-z0-9_]+)\s*\(", text)))


def test_library_file_is_sm100a_cubin():
    path = _lib.LIB_PATH
    assert os.path.exists(path), "build the library first (__graft_entry__.build())"
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_exports_every_declared_symbol():
    lib = _lib.load()
    declared = declared_functions()
    assert set(declared) == set(_lib.EXPORTS), f"header vs binding mismatch: {declared} vs {_lib.EXPORTS}"
    for name in declared:
        assert hasattr(lib, name), f"{name} not exported"


def test_version_and_workspace_formula():
    lib = _lib.load()
    assert lib.rs_version() >= 10300
    ws = lib.rs_workspace_bytes(4096, 4096, 192, 0, 0, 0)
    # two sweep partitions x 192 sweeps x 457 blocks x 9 waves of 16 B records
    # (standard form) + the same with 5 scale records per block (scaled form),
    # + 64 tiles (2 rows per lane) x 192 progress flags + the per-unit range words
    # ([2][k+1] u32: scaled form safe per sweep partition and unit) + trash slot
    nblk = (4096 + 8) // 9 + 1
    coef = -(-2 * 192 * nblk * 9 * 16 // 256) * 256
    scaled = -(-2 * 192 * nblk * 14 * 16 // 256) * 256
    flags = -(-(64 * 192 + 1) * 4 // 256) * 256
    trash = 32 * 4 * 8  # one slot per lane for the widest tile (fp32: 4 rows per lane)
    unsafe = -(-2 * (192 + 1) * 4 // 256) * 256
    assert ws == coef + scaled + flags + unsafe + trash
    assert ws % 256 == 0
    assert lib.rs_workspace_bytes(4096, 4096, 192, 0, 1, 0) > ws  # reflector records are 32 B
    # fp32: the same 16-byte record blocks (paired rotations; reflector (s, d, e, pad)) with
    # 3 scale records per block (9 fp32 scales); a build with the optional 16-sweep window
    # (RS_F32_WIDE=1) uses 17-column blocks with 5 scale records on the right side
    ws32 = coef + -(-2 * 192 * nblk * 12 * 16 // 256) * 256 + flags + unsafe + trash
    nblk16 = (4096 + 16) // 17 + 1
    ws32w = (-(-2 * 192 * nblk16 * 17 * 16 // 256) * 256 + -(-2 * 192 * nblk16 * 22 * 16 // 256) * 256
             + flags + unsafe + trash)
    assert lib.rs_workspace_bytes(4096, 4096, 192, 0, 0, 1) in (ws32, ws32w)
    assert lib.rs_workspace_bytes(4096, 4096, 192, 0, 1, 1) == lib.rs_workspace_bytes(4096, 4096, 192, 0, 0, 1)
    assert lib.rs_workspace_bytes(4096, 4096, 192, 1, 0, 1) == ws32  # left side: 8-sweep window
    assert lib.rs_workspace_bytes(4096, 1, 4, 0, 0, 0) == 0       # invalid: n < 2


@pytest.mark.parametrize("args,msg", [
    (dict(m=4, n=1), "at least 2 columns"),
    (dict(side=1, m=1), "at least 2 rows"),
    (dict(lda=2), "lda"),
    (dict(ldcs=1), "ldcs"),
    (dict(k=0), "k >= 1"),
    (dict(side=7), "side"),
    (dict(order=3), "order"),
    (dict(kind=9), "kind"),
])
def test_argument_errors_return_einval(args, msg):
    lib = _lib.load()
    p = dict(m=4, n=6, lda=4, ldcs=5, k=2, side=0, order=0, kind=0)
    p.update(args)
    dummy = ctypes.c_void_p(16)
    st = lib.rs_apply_f64(dummy, p["m"], p["n"], p["lda"], dummy, dummy, p["ldcs"], p["k"], p["side"],
                          p["order"], p["kind"], 1, None, 0, None)
    assert st == _lib.RS_EINVAL
    assert msg in _lib.last_error()
    with pytest.raises(ValueError, match=msg):
        _lib.check(st, "rs_apply_f64")


def test_zero_rows_ok_without_gpu():
    lib = _lib.load()
    assert lib.rs_apply_f64(None, 0, 6, 1, None, None, 5, 2, 0, 0, 0, 1, None, 0, None) == _lib.RS_OK


def test_packed_mode_requires_workspace():
    lib = _lib.load()
    dummy = ctypes.c_void_p(16)
    st = lib.rs_pack_f64(dummy, dummy, 5, 4, 6, 2, 0, 0, 0, None, 0, None)
    assert st == _lib.RS_EINVAL and "workspace" in _lib.last_error()


def test_last_error_is_thread_local():
    import threading

    lib = _lib.load()
    lib.rs_apply_f64(None, 4, 1, 4, None, None, 5, 2, 0, 0, 0, 1, None, 0, None)
    seen = {}

    def other():
        seen["msg"] = _lib.last_error()

    t = threading.Thread(target=other)
    t.start()
    t.join()
    assert seen["msg"] == ""
    assert "columns" in _lib.last_error()


def test_library_does_not_link_the_oracle():
    out = subprocess.run(["nm", "-D", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle_" not in out
