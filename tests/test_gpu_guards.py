"""Out-of-bounds write detection without compute-sanitizer (closed on this GPU pool).

Every buffer the library touches is embedded in a larger allocation whose surroundings are
filled with a signalling-NaN canary bit pattern: A as a row-block view (lda > m, the rows
above and below and the columns past n are canaries), C/S (must also stay bit-identical:
the library only reads them), the caller workspace (canaries past rs_workspace_bytes) and
the host matrix of the streaming entry point. After each call every canary must be intact
and the result must equal the oracle (strict: bitwise; fast: 10*k*eps). Cases cover the
forced multi-round / multi-CTA geometries (ring hand-offs, flags, trash slots for rows past
the matrix), both sides, orders and kinds, the micro-kernel API and the DMMA variant.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import assert_bitwise

pytestmark = pytest.mark.gpu

CANARY = np.uint64(0x7FF4DEADBEEF1234)  # a signalling NaN no kernel produces


def _canaried(shape, rows_pad=5, cols_pad=3, lead=13):
    """A column-major float64 view of `shape` inside a canary-filled device buffer."""
    import torch

    m, n = shape
    lda = m + 2 * rows_pad
    total = lead + lda * (n + cols_pad) + 64
    buf = torch.empty(total, dtype=torch.float64, device="cuda")
    buf.view(torch.int64).fill_(int(np.int64(CANARY.astype(np.int64))))
    view = buf[lead + rows_pad:lead + rows_pad + lda * n].as_strided((m, n), (1, lda)) if n > 0 else None
    return buf, view


def _canaries_intact(buf, view_mask):
    import torch

    bits = buf.view(torch.int64).cpu().numpy().view(np.uint64)
    outside = bits[~view_mask]
    return bool(np.all(outside == CANARY)), int(np.sum(outside != CANARY))


def _mask_for(buf, view):
    mask = np.zeros(buf.numel(), dtype=bool)
    base = view.storage_offset()
    m, n = view.shape
    lda = view.stride(1)
    for j in range(n):
        mask[base + j * lda: base + j * lda + m] = True
    return mask


CASES = [
    (100, 50, 40, "right", "forward", "rotation"),
    (90, 60, 41, "left", "reverse", "reflector"),
    (129, 130, 20, "left", "forward", "rotation"),
    (300, 37, 33, "right", "reverse", "reflector"),
    (65, 9, 8, "right", "forward", "rotation"),
]


@pytest.mark.parametrize("geom", [("", ""), ("1", ""), ("4", "3"), ("2", "5")])
def test_no_writes_outside_buffers(cuda, oracle_mod, monkeypatch, geom):
    import torch

    from paper_2412_01852_b200 import apply_device, compare, generate_sequence, make_inputs, workspace_bytes

    mw, grid = geom
    for key, val in (("RS_DEBUG_MAX_WARPS", mw), ("RS_DEBUG_GRID", grid)):
        if val:
            monkeypatch.setenv(key, val)
        else:
            monkeypatch.delenv(key, raising=False)
    for (m, n, k, side, order, kind) in CASES:
        A0, seq = make_inputs(m, n, k, 31)
        if side == "left":
            seq = generate_sequence(m, k, 32)
        C, S = seq.C.copy(order="F"), seq.S.copy(order="F")
        C[2, 1], S[2, 1] = 0.0, 1.0  # a per-unit fallback in fast mode
        ref = A0.copy(order="F")
        oracle_mod.apply_naive(ref, C, S, side=side, order=order, kind=kind)
        for fast in (False, True):
            buf, view = _canaried((m, n))
            view.copy_(torch.from_numpy(A0))
            mask = _mask_for(buf, view)
            cbuf, Cv = _canaried(C.shape)
            sbuf, Sv = _canaried(S.shape)
            Cv.copy_(torch.from_numpy(C))
            Sv.copy_(torch.from_numpy(S))
            cmask, smask = _mask_for(cbuf, Cv), _mask_for(sbuf, Sv)
            need = workspace_bytes(m, n, k, side=side, kind=kind)
            ws = torch.empty(need + 4096, dtype=torch.uint8, device="cuda")
            ws[need:].fill_(0xA5)
            apply_device(view, (Cv, Sv), kind=kind, fast=fast, side=side, order=order, workspace=ws[:need])
            torch.cuda.synchronize()
            tag = f"{m}x{n} k={k} {side}/{order}/{kind} fast={fast} geom={geom}"
            ok, bad = _canaries_intact(buf, mask)
            assert ok, f"{bad} canaries around A overwritten: {tag}"
            for b, mk, X in ((cbuf, cmask, C), (sbuf, smask, S)):
                assert _canaries_intact(b, mk)[0], f"C/S canaries overwritten: {tag}"
            assert_bitwise(C, Cv.cpu().numpy(), f"C modified: {tag}")
            assert_bitwise(S, Sv.cpu().numpy(), f"S modified: {tag}")
            assert bool((ws[need:] == 0xA5).all()), f"workspace overrun: {tag}"
            got = view.cpu().numpy()
            rep = compare(ref, got, "baseline" if fast else "strict", k=k)
            assert rep.passed, f"{tag}: {rep}"


def test_host_streaming_and_variants_no_overrun(cuda, oracle_mod):
    """The host-buffer entry point writes only the caller's matrix (host canaries around a
    row-block view); the micro-kernel API and the DMMA variant stay inside their buffers."""
    import torch

    from paper_2412_01852_b200 import apply_dmma, apply_host, compare, make_inputs
    from paper_2412_01852_b200.kernels import KernelShape, kernel_wave_apply

    for (m, n, k) in ((300, 257, 17), (64, 700, 40)):
        A0, seq = make_inputs(m, n, k, 5)
        ref = A0.copy(order="F")
        oracle_mod.apply_naive(ref, seq.C, seq.S)
        host = np.full((m + 9, n + 2), np.nan, order="F")
        host.view(np.uint64)[...] = CANARY
        view = host[4:4 + m, :n]
        view[...] = A0
        apply_host(view, seq, fast=False)
        assert_bitwise(ref, view, "host streaming")
        outside = np.ones(host.shape, dtype=bool)
        outside[4:4 + m, :n] = False
        assert np.all(host.view(np.uint64)[outside] == CANARY), "host canaries overwritten"
        # DMMA variant in a canaried device view
        buf, dview = _canaried((m, n))
        dview.copy_(torch.from_numpy(A0))
        mask = _mask_for(buf, dview)
        apply_dmma(dview, seq)
        torch.cuda.synchronize()
        assert _canaries_intact(buf, mask)[0], "DMMA variant wrote outside A"
        assert compare(ref, dview.cpu().numpy(), "baseline", k=k).passed
    # micro-kernel API: panel rows beyond m_r and columns beyond the waves untouched
    rng = np.random.Generator(np.random.Philox(3))
    P0 = np.ascontiguousarray(rng.standard_normal((30, 37)))
    th = rng.uniform(0, 2 * np.pi, size=10 * 5)
    dP = torch.from_numpy(P0).cuda()
    kernel_wave_apply(dP, np.cos(th), np.sin(th), 10, KernelShape(37, 5), "rotation", 4)
    P = dP.cpu().numpy()
    ref = P0.copy()
    oracle_mod.wave_apply(ref, np.cos(th), np.sin(th), 10, 5, 4)
    assert_bitwise(ref, P, "wave apply")
    assert_bitwise(P0[:4], P[:4], "columns before col0 untouched")
    assert_bitwise(P0[4 + 10 + 5:], P[4 + 10 + 5:], "columns past the waves untouched")
